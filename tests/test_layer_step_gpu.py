"""One SGD step of a 2-layer ReLU MLP built from the fused-epilogue kernels vs torch fp32 autograd."""

import pytest

torch = pytest.importorskip("torch")

from paper_1806_03377_b200 import _native as nat  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("B,din,dh,dout", [(32, 1024, 1024, 1024), (64, 256, 512, 128)])
def test_two_layer_step_fp32_matches_autograd(B, din, dh, dout):
    g = torch.Generator(device="cuda").manual_seed(0)
    X = torch.randn(B, din, device="cuda", generator=g)
    T = torch.randn(B, dout, device="cuda", generator=g)
    W1 = torch.randn(dh, din, device="cuda", generator=g) * (2 / din) ** 0.5
    b1 = torch.randn(dh, device="cuda", generator=g) * 0.01
    W2 = torch.randn(dout, dh, device="cuda", generator=g) * (2 / dh) ** 0.5
    b2 = torch.randn(dout, device="cuda", generator=g) * 0.01
    lr = 1e-3
    # torch reference
    p = [t.clone().requires_grad_(True) for t in (W1, b1, W2, b2)]
    h = torch.relu(X @ p[0].t() + p[1])
    z = h @ p[2].t() + p[3]
    loss = 0.5 / B * ((z - T) ** 2).sum()
    loss.backward()
    ref = [t.detach() - lr * t.grad for t in p]
    # kernels
    H = torch.empty(B, dh, device="cuda")
    dZ = torch.empty(B, dout, device="cuda")
    dH = torch.empty(B, dh, device="cuda")
    L = torch.zeros(1, device="cuda")
    nat.gemm(X, False, W1, False, B, dh, din, kind=nat.EPI_STORE, out=H, bias=b1, relu=True)
    nat.gemm(H, False, W2, False, B, dout, dh, kind=nat.EPI_LOSS, out=dZ, bias=b2, target=T, scale=1.0 / B, loss=L)
    nat.gemm(dZ, False, W2, True, B, dh, dout, kind=nat.EPI_MASK, out=dH, mask=H)
    m = [t.clone() for t in (W1, b1, W2, b2)]
    ring = [torch.empty_like(t) for t in m]
    nat.gemm(dZ, True, H, True, dout, dh, B, kind=nat.EPI_SGD, out=ring[2], master=m[2], lr=lr)
    nat.bias_sgd(dZ, B, dout, m[3], ring[3], lr)
    nat.gemm(dH, True, X, True, dh, din, B, kind=nat.EPI_SGD, out=ring[0], master=m[0], lr=lr)
    nat.bias_sgd(dH, B, dh, m[1], ring[1], lr)
    torch.cuda.synchronize()
    assert abs(float(L) - float(loss)) <= 1e-5 * float(loss)
    for got, want, init in zip(m, ref, (W1, b1, W2, b2)):
        delta_err = (got - want).norm() / (want - init).norm()
        assert delta_err <= 1e-4, float(delta_err)
