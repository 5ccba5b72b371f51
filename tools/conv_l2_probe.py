"""One VGG-16 conv layer pass (default: layer 2, 224x224, 64 -> 64, batch 32) launched a few
times, for ncu captures of the conv tile variants (PD_CONV_ROWS=0|1).
    python tools/conv_l2_probe.py [fwd|dgrad] [H] [cin] [cout]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_03377_b200 import _native as nat  # noqa: E402


def main():
    pas = sys.argv[1] if len(sys.argv) > 1 else "fwd"
    h = int(sys.argv[2]) if len(sys.argv) > 2 else 224
    ci = int(sys.argv[3]) if len(sys.argv) > 3 else 64
    co = int(sys.argv[4]) if len(sys.argv) > 4 else 64
    n = 32
    x = torch.randn(n, h, h, ci, device="cuda").bfloat16().relu()
    wt = (torch.randn(9 * ci, co, device="cuda") * 0.02).bfloat16()
    bias = torch.zeros(co, device="cuda")
    y = torch.empty(n, h, h, co, device="cuda", dtype=torch.bfloat16)
    dy = torch.randn(n, h, h, co, device="cuda").bfloat16()
    dx = torch.empty_like(x)
    for _ in range(3):
        if pas == "fwd":
            nat.conv3x3(nat.PD_CONV_FWD, x, wt, n, h, h, ci, co, out=y, bias=bias, relu=True)
        else:
            nat.conv3x3(nat.PD_CONV_DGRAD, dy, wt, n, h, h, ci, co, out=dx, mask=x)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
