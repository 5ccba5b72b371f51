"""GPT-2 head GEMM (8 x 1024 tokens x 1024 -> 50304 padded vocabulary, fp32 logits + bias) and the
softmax cross-entropy that reads them, CUDA events; torch.matmul with a bf16 output for reference."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
    T, d, V = 8192, 1024, 50304
    h = torch.randn(T, d, device="cuda").bfloat16()
    W = (torch.randn(V, d, device="cuda") / d ** 0.5).bfloat16()
    bias = torch.zeros(V, device="cuda")
    logits = torch.empty(T, V, device="cuda")
    fl = 2.0 * T * V * d
    ours = timeit(lambda: nat.gemm(h, False, W, False, T, V, d, kind=nat.EPI_GRADF32, out=logits, bias=bias))
    ref = timeit(lambda: torch.mm(h.float(), W.float().t(), out=logits)) if False else float("nan")
    ref_bf = timeit(lambda: torch.matmul(h, W.t()))
    labels = torch.randint(0, 50257, (T,), device="cuda", dtype=torch.int32)
    dz = torch.empty(T, V, device="cuda", dtype=torch.bfloat16)
    loss = torch.zeros(1, device="cuda")
    L = nat.lib()
    ce = timeit(lambda: L.pd_softmax_ce_vocab(nat.ptr(logits), V, nat.ptr(labels), T, 50257, V, nat.ptr(dz), V,
                                          nat.ptr(loss), nat.stream_ptr()))
    print(json.dumps({"softmax_ce_ms": round(ce, 4), "ce_gbs": round((T * V * 4 + T * V * 2) / ce / 1e6, 1)}))
    print(json.dumps({"head_fwd_ms": round(ours, 4), "tflops": round(fl / ours / 1e9, 1),
                      "torch_bf16_out_ms": round(ref_bf, 4), 
                      "logits_bytes": T * V * 4}))


if __name__ == "__main__":
    main()
