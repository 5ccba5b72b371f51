"""Attention fwd / bwd timing at GPT-2 medium shape (8 x 1024 tokens, 16 heads), CUDA events.

Algorithmic FLOPs (causal): fwd 2 * 2 * B*H*S^2*64 / 2, bwd 2.5x fwd.  Compared with torch SDPA.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_03377_b200 import _native as nat  # noqa: E402


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    B, S, H = 8, 1024, 16
    d = 64 * H
    qkv = torch.randn(B * S, 3 * d, device="cuda").bfloat16()
    out = torch.empty(B * S, d, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B, H, S, device="cuda")
    dout = torch.randn(B * S, d, device="cuda").bfloat16()
    dvec = torch.empty(B, H, S, device="cuda")
    dq = torch.empty(B * S, d, device="cuda")
    dqkv = torch.empty(B * S, 3 * d, device="cuda", dtype=torch.bfloat16)
    L = nat.lib()
    st = nat.stream_ptr()
    fwd = lambda: L.pd_attention_fwd(nat.ptr(qkv), nat.ptr(out), nat.ptr(lse), B, S, H, st)  # noqa: E731
    bwd = lambda: L.pd_attention_bwd(nat.ptr(qkv), nat.ptr(out), nat.ptr(dout), nat.ptr(lse), nat.ptr(dvec),  # noqa
                                     nat.ptr(dq), nat.ptr(dqkv), B, S, H, st)
    t_f = timeit(fwd)
    t_b = timeit(bwd)
    q, k, v = (t.reshape(B, S, H, 64).transpose(1, 2) for t in qkv.view(B, S, 3 * d).split(d, dim=-1))
    t_t = timeit(lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True))
    ff = 2.0 * 2 * B * H * S * S * 64 / 2
    print(json.dumps({"fwd_ms": round(t_f, 4), "bwd_ms": round(t_b, 4), "torch_sdpa_fwd_ms": round(t_t, 4),
                      "fwd_tflops": round(ff / t_f / 1e9, 1), "bwd_tflops": round(2.5 * ff / t_b / 1e9, 1),
                      "torch_sdpa_fwd_tflops": round(ff / t_t / 1e9, 1)}))


if __name__ == "__main__":
    main()
