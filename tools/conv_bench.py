"""Per-layer timing of the VGG-16 convolution passes at minibatch 32 (CUDA events, warm).

For every conv layer: implicit-GEMM forward, dgrad, split-K wgrad (+ the fixed-order reduction),
and cuDNN (torch, channels_last bf16) forward for comparison.  Prints one JSON line per layer.
    python tools/conv_bench.py [batch]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_03377_b200 import _native as nat  # noqa: E402
from paper_1806_03377_b200.models import vgg16  # noqa: E402


def timeit(fn, reps=10):
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
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    spec = vgg16(batch=B)
    tot = {"fwd": 0.0, "dgrad": 0.0, "wgrad": 0.0, "cudnn_fwd": 0.0}
    for i, g in enumerate(spec.geoms()):
        if g.kind != "conv" or g.im2col:
            continue
        n, h, w, ci, co = B, g.h, g.w, g.c_in, g.c_out
        x = torch.randn(n, h, w, ci, device="cuda").bfloat16().relu()
        wt = (torch.randn(9 * ci, co, device="cuda") * 0.02).bfloat16()
        bias = torch.zeros(co, device="cuda")
        y = torch.empty(n, h, w, co, device="cuda", dtype=torch.bfloat16)
        dy = torch.randn(n, h, w, co, device="cuda").bfloat16()
        dx = torch.empty_like(x)
        S = nat.splitk_plan(9 * ci, co, n * h * w)
        part = torch.empty(S, 9 * ci, co, device="cuda")
        master = torch.zeros(9 * ci, co, device="cuda")
        ring = torch.empty(9 * ci, co, device="cuda", dtype=torch.bfloat16)
        flops = 2.0 * n * h * w * 9 * ci * co
        t_f = timeit(lambda: nat.conv3x3(nat.PD_CONV_FWD, x, wt, n, h, w, ci, co, out=y, bias=bias, relu=True))
        t_d = timeit(lambda: nat.conv3x3(nat.PD_CONV_DGRAD, dy, wt, n, h, w, ci, co, out=dx, mask=x))

        def wg():
            nat.conv3x3(nat.PD_CONV_WGRAD, x, dy, n, h, w, ci, co, out=part)
            nat.check(nat.lib().pd_reduce_sgd(nat.PD_BF16, nat.ptr(part), S, 9 * ci * co, 9 * ci * co, None,
                                              nat.ptr(master), nat.ptr(ring), 0.0, nat.stream_ptr()), "reduce")
        t_w = timeit(wg)
        xt = x.permute(0, 3, 1, 2)  # channels_last view
        wc = wt.view(3, 3, ci, co).permute(3, 2, 0, 1).contiguous(memory_format=torch.channels_last)
        t_c = timeit(lambda: torch.nn.functional.conv2d(xt, wc, padding=1))
        for k, v in (("fwd", t_f), ("dgrad", t_d), ("wgrad", t_w), ("cudnn_fwd", t_c)):
            tot[k] += v
        print(json.dumps({"layer": i + 1, "hw": h, "cin": ci, "cout": co, "splits": S,
                          "fwd_ms": round(t_f, 4), "dgrad_ms": round(t_d, 4), "wgrad_ms": round(t_w, 4),
                          "cudnn_fwd_ms": round(t_c, 4), "fwd_tflops": round(flops / t_f / 1e9, 1),
                          "dgrad_tflops": round(flops / t_d / 1e9, 1), "wgrad_tflops": round(flops / t_w / 1e9, 1),
                          "cudnn_fwd_tflops": round(flops / t_c / 1e9, 1)}), flush=True)
    print(json.dumps({"total_ms": {k: round(v, 3) for k, v in tot.items()}}))


if __name__ == "__main__":
    main()
