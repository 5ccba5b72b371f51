"""Diagnostic: per-tile event timeline of the attention backward main kernel (a -DPD_ATTN_TRACE=1
build loaded with PD_LIB).  Phases per query tile n of a key-tile CTA: wait for S^T/dP^T (sdp_full),
exp / dS math until sdp_free, wait for the previous tile's dV/dK/dQ MMAs (dq_full), dQ flush + P / dS
stores until pds_ready."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_03377_b200 import _native as nat  # noqa: E402


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
    L.pd_attention_fwd(nat.ptr(qkv), nat.ptr(out), nat.ptr(lse), B, S, H, st)
    bwd = lambda: L.pd_attention_bwd(nat.ptr(qkv), nat.ptr(out), nat.ptr(dout), nat.ptr(lse), nat.ptr(dvec),  # noqa
                                     nat.ptr(dq), nat.ptr(dqkv), B, S, H, st)
    for _ in range(3):
        bwd()
    torch.cuda.synchronize()
    L.pd_attn_trace_clear()
    bwd()
    torch.cuda.synchronize()
    n = min(148, H * B * (S // 128))  # persistent kernel: one CTA per SM, stamps for its first 9 tiles
    buf = (ctypes.c_ulonglong * (2048 * 64))()
    L.pd_attn_trace(buf, n)
    t = np.frombuffer(buf, dtype=np.uint64).reshape(2048, 64)[:n].astype(np.int64)
    f = lambda a: round(float(np.mean(a)) / 1e3, 3)  # noqa: E731
    ph = {"first_s_after_start": [], "wait_sdp": [], "math": [], "wait_dq": [], "stage_store": []}
    for c in range(n):
        ph["first_s_after_start"].append(t[c, 1] - t[c, 0])
        for g in range(1, 9):
            ph["wait_sdp"].append(t[c, 1 + 4 * g] - t[c, 4 + 4 * (g - 1)])
            ph["math"].append(t[c, 2 + 4 * g] - t[c, 1 + 4 * g])
            ph["wait_dq"].append(t[c, 3 + 4 * g] - t[c, 2 + 4 * g])
            ph["stage_store"].append(t[c, 4 + 4 * g] - t[c, 3 + 4 * g])
    res = {k: f(v) for k, v in ph.items()}
    res["per_tile_us"] = f([(t[c, 4 + 4 * 8] - t[c, 4]) / 8 for c in range(n)])
    res["kernel_span_us"] = float((t[:, 41].max() - t[:, 0].min()) / 1e3)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
