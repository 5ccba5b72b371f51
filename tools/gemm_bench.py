"""Time the three stage GEMMs of one MLP-8192 layer (fwd / dgrad / wgrad+SGD) with CUDA events."""
import json
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_1806_03377_b200 import _native as nat  # noqa: E402


def timeit(fn, iters=10, warm=3):
    for _ in range(warm):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    B = int(args[0]) if len(args) > 0 else 2048
    D = int(args[1]) if len(args) > 1 else 8192
    bf = torch.bfloat16
    X = torch.randn(B, D, device="cuda").to(bf)
    W = (torch.randn(D, D, device="cuda") / D ** 0.5).to(bf)
    dZ = torch.randn(B, D, device="cuda").to(bf)
    Y = torch.empty(B, D, device="cuda", dtype=bf)
    bias = torch.zeros(D, device="cuda")
    master = W.float()
    ring = torch.empty(D, D, device="cuda", dtype=bf)
    flops = 2.0 * B * D * D
    res = {}
    res["fwd_ms"] = timeit(lambda: nat.gemm(X, False, W, False, B, D, D, kind=nat.EPI_STORE, out=Y, bias=bias, relu=True))
    res["dgrad_ms"] = timeit(lambda: nat.gemm(dZ, False, W, True, B, D, D, kind=nat.EPI_MASK, out=Y, mask=X))
    res["wgrad_sgd_ms"] = timeit(lambda: nat.gemm(dZ, True, X, True, D, D, B, kind=nat.EPI_SGD, out=ring, master=master, lr=1e-6))
    res["torch_mm_ms"] = timeit(lambda: torch.matmul(X, W.t()))
    if "--wgrad-variants" in sys.argv:
        Wb = torch.empty(D, D, device="cuda", dtype=bf)
        G = torch.empty(D, D, device="cuda")
        res["wgrad_store_bf16_ms"] = timeit(lambda: nat.gemm(dZ, True, X, True, D, D, B, kind=nat.EPI_STORE, out=Wb))
        res["wgrad_gradf32_ms"] = timeit(lambda: nat.gemm(dZ, True, X, True, D, D, B, kind=nat.EPI_GRADF32, out=G))
        res["copy_fp32_1GB_ms"] = timeit(lambda: G.copy_(master))
    for k in list(res):
        res[k.replace("_ms", "_tflops")] = flops / (res[k] * 1e-3) / 1e12
    res["B"], res["D"] = B, D
    print(json.dumps(res))


if __name__ == "__main__":
    main()
