"""Convolutional-stage kernels (configs[2], VGG-16) against torch fp32 on the same bf16 inputs.

Implicit-GEMM 3x3 convolution (TMA im2col) forward / dgrad / split-K wgrad, the first-layer im2col,
max pool with argmax, tall bias gradients, split-K reduce + SGD and softmax cross-entropy.
Tolerance: outputs are bf16 (8-bit mantissa) from fp32 accumulation, so every comparison is
|got - want| <= 1.5e-2 * max|want| (+ a small absolute floor); fp32 outputs (wgrad partials,
losses) use 2e-3 relative.
"""
import pytest
import torch

from paper_1806_03377_b200 import _native as nat

pytestmark = pytest.mark.gpu

F = torch.nn.functional


def _close(got, want, rel=1.5e-2, floor=1e-3):
    got, want = got.float(), want.float()
    err = (got - want).abs().max().item()
    scale = want.abs().max().item()
    assert err <= rel * scale + floor, f"max err {err:.3e} vs scale {scale:.3e}"


def _wt_to_oihw(wt, cin, cout):
    # Wt[(r*3+s)*cin + c][cout] -> torch weight [cout, cin, 3, 3]
    return wt.float().view(3, 3, cin, cout).permute(3, 2, 0, 1).contiguous()


SHAPES = [(2, 8, 8, 64, 128), (1, 7, 7, 64, 64), (2, 14, 14, 128, 64), (2, 16, 16, 256, 256), (1, 28, 28, 64, 512)]
# wide and ragged images: 128-pixel tiles straddling image rows and images (W 112, 120, 224, 250),
# an odd tile count (a CTA pair's padding tile), a partial last tile
ROW_SHAPES = [(1, 5, 112, 64, 64), (2, 3, 224, 64, 128), (1, 4, 120, 128, 64), (1, 3, 250, 64, 256),
              (2, 6, 56, 64, 64)]


@pytest.mark.parametrize("n,h,w,cin,cout", SHAPES + ROW_SHAPES)
def test_conv_fwd(n, h, w, cin, cout):
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(n, h, w, cin, device="cuda", generator=g).bfloat16()
    wt = (torch.randn(9 * cin, cout, device="cuda", generator=g) / (3 * cin ** 0.5)).bfloat16()
    bias = torch.randn(cout, device="cuda", generator=g) * 0.1
    y = torch.empty(n, h, w, cout, device="cuda", dtype=torch.bfloat16)
    nat.conv3x3(nat.PD_CONV_FWD, x, wt, n, h, w, cin, cout, out=y, bias=bias, relu=True)
    torch.cuda.synchronize()
    ref = F.relu(F.conv2d(x.float().permute(0, 3, 1, 2), _wt_to_oihw(wt, cin, cout), bias, padding=1))
    _close(y, ref.permute(0, 2, 3, 1))


@pytest.mark.parametrize("n,h,w,cin,cout", SHAPES + ROW_SHAPES)
def test_conv_dgrad(n, h, w, cin, cout):
    g = torch.Generator(device="cuda").manual_seed(2)
    dy = torch.randn(n, h, w, cout, device="cuda", generator=g).bfloat16()
    wt = (torch.randn(9 * cin, cout, device="cuda", generator=g) / (3 * cout ** 0.5)).bfloat16()
    x = F.relu(torch.randn(n, h, w, cin, device="cuda", generator=g)).bfloat16()  # post-ReLU layer input
    dx = torch.empty(n, h, w, cin, device="cuda", dtype=torch.bfloat16)
    nat.conv3x3(nat.PD_CONV_DGRAD, dy, wt, n, h, w, cin, cout, out=dx, mask=x)
    torch.cuda.synchronize()
    ref = torch.nn.grad.conv2d_input((n, cin, h, w), _wt_to_oihw(wt, cin, cout), dy.float().permute(0, 3, 1, 2),
                                     padding=1)
    ref = ref.permute(0, 2, 3, 1) * (x.float() > 0)
    _close(dx, ref)


@pytest.mark.parametrize("n,h,w,cin,cout", SHAPES)
def test_conv_wgrad_splitk(n, h, w, cin, cout):
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(n, h, w, cin, device="cuda", generator=g).bfloat16()
    dy = torch.randn(n, h, w, cout, device="cuda", generator=g).bfloat16()
    S = nat.splitk_plan(9 * cin, cout, n * h * w)
    part = torch.full((S, 9 * cin, cout), float("nan"), device="cuda")
    nat.conv3x3(nat.PD_CONV_WGRAD, x, dy, n, h, w, cin, cout, out=part)
    # fold the partials with the SGD reduction: master = 0 - 1.0 * sum
    master = torch.zeros(9 * cin, cout, device="cuda")
    ring = torch.empty(9 * cin, cout, device="cuda", dtype=torch.bfloat16)
    nat.check(nat.lib().pd_reduce_sgd(nat.PD_BF16, nat.ptr(part), S, 9 * cin * cout, 9 * cin * cout, None,
                                      nat.ptr(master), nat.ptr(ring), 1.0, nat.stream_ptr()), "reduce")
    torch.cuda.synchronize()
    ref = torch.nn.grad.conv2d_weight(x.float().permute(0, 3, 1, 2), (cout, cin, 3, 3),
                                      dy.float().permute(0, 3, 1, 2), padding=1)
    ref_wt = ref.permute(2, 3, 1, 0).reshape(9 * cin, cout)
    _close(-master, ref_wt, rel=2e-3)
    _close(ring, -ref_wt)


def test_first_layer_im2col_gemm():
    n, h, w, c, cout = 2, 16, 16, 3, 64
    g = torch.Generator(device="cuda").manual_seed(4)
    x = torch.randn(n, h, w, c, device="cuda", generator=g).bfloat16()
    cols = torch.empty(n * h * w, 64, device="cuda", dtype=torch.bfloat16)
    nat.check(nat.lib().pd_im2col3(nat.ptr(x), nat.ptr(cols), n, h, w, c, 64, nat.stream_ptr()), "im2col")
    wt = torch.zeros(64, cout, device="cuda")
    wt[:27] = torch.randn(27, cout, device="cuda", generator=g) * 0.2
    wt = wt.bfloat16()
    bias = torch.randn(cout, device="cuda", generator=g) * 0.1
    y = torch.empty(n * h * w, cout, device="cuda", dtype=torch.bfloat16)
    nat.gemm(cols, False, wt, True, n * h * w, cout, 64, out=y, bias=bias, relu=True)
    torch.cuda.synchronize()
    ref = F.relu(F.conv2d(x.float().permute(0, 3, 1, 2), _wt_to_oihw(wt[:27].contiguous(), c, cout), bias, padding=1))
    _close(y.view(n, h, w, cout), ref.permute(0, 2, 3, 1))
    # wgrad of the im2col'ed layer: split-K plain GEMM over the pixel rows
    dy = torch.randn(n * h * w, cout, device="cuda", generator=g).bfloat16()
    S = nat.splitk_plan(64, cout, n * h * w)
    part = torch.empty(S, 64, cout, device="cuda")
    nat.conv3x3(nat.PD_GEMM_WGRAD_SPLITK, cols, dy, n, h, w, 64, cout, out=part)
    torch.cuda.synchronize()
    ref_w = cols.float().t() @ dy.float()
    _close(part.sum(0), ref_w, rel=2e-3)


@pytest.mark.parametrize("n,h,w,c", [(2, 8, 8, 64), (3, 14, 14, 128), (1, 224, 224, 64)])
def test_maxpool(n, h, w, c):
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(n, h, w, c, device="cuda", generator=g).bfloat16()
    y = torch.empty(n, h // 2, w // 2, c, device="cuda", dtype=torch.bfloat16)
    arg = torch.empty(n, h // 2, w // 2, c, device="cuda", dtype=torch.uint8)
    nat.check(nat.lib().pd_maxpool2(nat.ptr(x), nat.ptr(y), nat.ptr(arg), n, h, w, c, nat.stream_ptr()), "pool")
    win = x.view(n, h // 2, 2, w // 2, 2, c).permute(0, 1, 3, 5, 2, 4).reshape(n, h // 2, w // 2, c, 4)
    want_v, want_i = win.float().max(-1)
    torch.cuda.synchronize()
    assert torch.equal(y.float(), want_v)
    first = (win.float() == want_v.unsqueeze(-1)).float().argmax(-1)  # first maximum in scan order
    assert torch.equal(arg.long(), first)
    dy = torch.randn(n, h // 2, w // 2, c, device="cuda", generator=g).bfloat16()
    dx = torch.full((n, h, w, c), 7.0, device="cuda", dtype=torch.bfloat16)
    nat.check(nat.lib().pd_maxpool2_bwd(nat.ptr(dy), nat.ptr(arg), nat.ptr(dx), n, h, w, c, nat.stream_ptr()), "bwd")
    want = torch.zeros(n, h // 2, w // 2, c, 4, device="cuda")
    want.scatter_(-1, first.unsqueeze(-1), dy.float().unsqueeze(-1))
    want = want.view(n, h // 2, w // 2, c, 2, 2).permute(0, 1, 4, 2, 5, 3).reshape(n, h, w, c)
    torch.cuda.synchronize()
    assert torch.equal(dx.float(), want)


@pytest.mark.parametrize("rows,c", [(1000, 64), (32 * 224 * 224, 64), (6272, 512), (33, 128)])
def test_bias_grad_tall(rows, c):
    g = torch.Generator(device="cuda").manual_seed(6)
    dz = torch.randn(rows, c, device="cuda", generator=g).bfloat16()
    nb = nat.lib().pd_colsum_blocks(rows, c)
    part = torch.empty(nb, c, device="cuda")
    grad = torch.empty(c, device="cuda")
    nat.check(nat.lib().pd_bias_grad_tall(nat.ptr(dz), rows, c, nat.ptr(part), nat.ptr(grad), None, None, 0.0,
                                          nat.stream_ptr()), "bias grad")
    torch.cuda.synchronize()
    ref = dz.double().sum(0)
    assert (grad.double() - ref).abs().max().item() <= 1e-4 * rows ** 0.5 + 1e-3
    # SGD form
    master = torch.ones(c, device="cuda")
    out = torch.empty(c, device="cuda")
    nat.check(nat.lib().pd_bias_grad_tall(nat.ptr(dz), rows, c, nat.ptr(part), None, nat.ptr(master), nat.ptr(out),
                                          0.5, nat.stream_ptr()), "bias sgd")
    torch.cuda.synchronize()
    assert torch.allclose(master, 1 - 0.5 * grad, atol=1e-5) and torch.equal(master, out)


def test_softmax_ce():
    B, V = 32, 1000
    g = torch.Generator(device="cuda").manual_seed(7)
    z = torch.randn(B, V, device="cuda", generator=g) * 3
    lab = torch.randint(0, V, (B,), device="cuda", generator=g, dtype=torch.int32)
    dz = torch.empty(B, V, device="cuda", dtype=torch.bfloat16)
    loss = torch.zeros(1, device="cuda")
    nat.check(nat.lib().pd_softmax_ce(nat.ptr(z), V, nat.ptr(lab), B, V, nat.ptr(dz), V, nat.ptr(loss),
                                      nat.stream_ptr()), "ce")
    zz = z.clone().requires_grad_(True)
    ref = F.cross_entropy(zz, lab.long())
    ref.backward()
    torch.cuda.synchronize()
    assert abs(loss.item() - ref.item()) <= 2e-3 * ref.item()
    _close(dz, zz.grad)
