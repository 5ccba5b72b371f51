"""Time every GEMM of one GPT-2 medium block (8 x 1024 tokens) with CUDA events, vs torch.matmul.

Shapes (T = 8192 tokens, d = 1024, f = 4096): forward qkv / out-proj / FC1 / FC2, their dgrads
(B operand MN-major) and wgrads (+ fused SGD).  One JSON line per GEMM.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_03377_b200 import _native as nat  # noqa: E402


def timeit(fn, iters=20, warm=3):
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
    T, d, f = 8192, 1024, 4096
    bf = torch.bfloat16
    total = {"ours": 0.0, "torch": 0.0}
    for name, N, K in (("qkv", 3 * d, d), ("proj", d, d), ("fc1", f, d), ("fc2", d, f)):
        X = torch.randn(T, K, device="cuda").to(bf)
        W = (torch.randn(N, K, device="cuda") / K ** 0.5).to(bf)
        Y = torch.empty(T, N, device="cuda", dtype=bf)
        dY = torch.randn(T, N, device="cuda").to(bf)
        dX = torch.empty(T, K, device="cuda", dtype=bf)
        master = W.float()
        ring = torch.empty(N, K, device="cuda", dtype=bf)
        bias = torch.zeros(N, device="cuda")
        fl = 2.0 * T * N * K
        rows = {
            "fwd": (timeit(lambda: nat.gemm(X, False, W, False, T, N, K, kind=nat.EPI_STORE, out=Y, bias=bias)),
                    timeit(lambda: torch.matmul(X, W.t()))),
            "dgrad": (timeit(lambda: nat.gemm(dY, False, W, True, T, K, N, kind=nat.EPI_STORE, out=dX)),
                      timeit(lambda: torch.matmul(dY, W))),
            "wgrad_sgd": (timeit(lambda: nat.gemm(dY, True, X, True, N, K, T, kind=nat.EPI_SGD, out=ring, master=master,
                                                  lr=0.0)),
                          timeit(lambda: torch.matmul(dY.t(), X))),
        }
        # the epilogues the pipeline actually runs (GELU fc1 stores pre-activation + output; proj / fc2
        # add the residual; the fc2 dgrad applies GELU'); compared with the plain-store rows above
        Z = torch.empty(T, N, device="cuda", dtype=bf)
        R = torch.randn(T, N, device="cuda").to(bf)
        if name == "fc1":
            epi = timeit(lambda: nat.gemm(X, False, W, False, T, N, K, kind=nat.EPI_GELU, out=Y, aux=Z, bias=bias))
            print(json.dumps({"gemm": name, "pass": "fwd+gelu", "ms": round(epi, 4), "tflops": round(fl / epi / 1e9, 1)}))
        if name in ("proj", "fc2"):
            epi = timeit(lambda: nat.gemm(X, False, W, False, T, N, K, kind=nat.EPI_RESID, out=Y, mask=R, bias=bias))
            print(json.dumps({"gemm": name, "pass": "fwd+resid", "ms": round(epi, 4), "tflops": round(fl / epi / 1e9, 1)}))
        if name == "fc2":
            Zf = torch.randn(T, K, device="cuda").to(bf)
            epi = timeit(lambda: nat.gemm(dY, False, W, True, T, K, N, kind=nat.EPI_GELU_BWD, out=dX, mask=Zf))
            print(json.dumps({"gemm": name, "pass": "dgrad+gelu'", "ms": round(epi, 4), "tflops": round(fl / epi / 1e9, 1)}))
        for pas, (a, b) in rows.items():
            total["ours"] += a
            total["torch"] += b
            print(json.dumps({"gemm": name, "pass": pas, "M": T if pas != "wgrad_sgd" else N,
                              "N": N if pas == "fwd" else K, "K": K if pas == "fwd" else (N if pas == "dgrad" else T),
                              "ms": round(a, 4), "tflops": round(fl / a / 1e9, 1),
                              "torch_ms": round(b, 4), "torch_tflops": round(fl / b / 1e9, 1)}), flush=True)
    print(json.dumps({"block_total_ms": {k: round(v, 4) for k, v in total.items()}}))


if __name__ == "__main__":
    main()
