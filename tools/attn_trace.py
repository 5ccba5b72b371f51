"""Diagnostic: per-tile event timeline of the attention forward (needs a -DPD_ATTN_TRACE=1 build,
loaded with PD_LIB).  Prints per-phase averages: prologue, s_full waits, softmax, o_done waits."""
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
    L = nat.lib()
    st = nat.stream_ptr()
    for _ in range(3):
        L.pd_attention_fwd(nat.ptr(qkv), nat.ptr(out), nat.ptr(lse), B, S, H, st)
    torch.cuda.synchronize()
    L.pd_attn_trace_clear()
    L.pd_attention_fwd(nat.ptr(qkv), nat.ptr(out), nat.ptr(lse), B, S, H, st)
    torch.cuda.synchronize()
    n = H * B * (S // 128)
    buf = (ctypes.c_ulonglong * (2048 * 64))()
    L.pd_attn_trace(buf, n)
    t = np.frombuffer(buf, dtype=np.uint64).reshape(2048, 64)[:n].astype(np.int64)
    t0 = t[:, 0].min()
    res = {"kernel_span_us": float((t[:, 41].max() - t0) / 1e3)}
    qt = np.array([7 - (c // (H * B)) for c in range(n)])
    pro, sw, sm, ow, tail = [], [], [], [], []
    for c in range(n):
        k = qt[c] + 1
        pro.append(t[c, 2] - t[c, 0])
        for j in range(k):
            if j > 0:
                sw.append(t[c, 2 + 4 * j] - t[c, 5 + 4 * (j - 1)])
            sm.append(t[c, 3 + 4 * j] - t[c, 2 + 4 * j])
            ow.append(t[c, 4 + 4 * j] - t[c, 3 + 4 * j])
            sm.append(t[c, 5 + 4 * j] - t[c, 4 + 4 * j])
        tail.append(t[c, 41] - t[c, 5 + 4 * (k - 1)])
    f = lambda a: round(float(np.mean(a)) / 1e3, 3)  # noqa: E731
    res.update({"prologue_to_first_s_us": f(pro), "s_full_wait_us": f(sw), "softmax_phase_us": f(sm),
                "o_done_wait_us": f(ow), "epilogue_us": f(tail)})
    per_tile = [(t[c, 5 + 4 * qt[c]] - t[c, 2]) / (qt[c] + 1) for c in range(n)]
    res["per_tile_us"] = f(per_tile)
    res["cta_span_us"] = f([t[c, 41] - t[c, 0] for c in range(n)])
    sms = t[:, 63]
    res["ctas_per_sm_max"] = int(np.bincount(sms.astype(np.int64)).max())
    print(json.dumps(res))
    np.save("gpurun_out/attn_trace.npy", t)


if __name__ == "__main__":
    main()
