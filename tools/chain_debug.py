"""Plain SGD of an L-layer ReLU MLP: kernels called from Python in the runtime's pattern vs torch autograd."""
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_1806_03377_b200 import _native as nat  # noqa: E402


def main(L=4, w=1024, B=32, steps=6, lr=2e-4):
    g = torch.Generator(device="cuda").manual_seed(0)
    Ws = [torch.randn(w, w, device="cuda", generator=g) * (2 / w) ** 0.5 for _ in range(L)]
    bs = [torch.randn(w, device="cuda", generator=g) * 0.01 for _ in range(L)]
    Xs = [torch.randn(B, w, device="cuda", generator=g) for _ in range(steps)]
    Ts = [torch.randn(B, w, device="cuda", generator=g) for _ in range(steps)]
    # torch
    P = [t.clone() for t in Ws] + [t.clone() for t in bs]
    ref_losses = []
    for s in range(steps):
        p = [t.clone().requires_grad_(True) for t in P]
        h = Xs[s]
        for l in range(L):
            z = h @ p[l].t() + p[L + l]
            h = torch.relu(z) if l < L - 1 else z
        loss = 0.5 / B * ((z - Ts[s]) ** 2).sum()
        loss.backward()
        ref_losses.append(float(loss))
        P = [t.detach() - lr * t.grad for t in p]
    # kernels
    mW = [t.clone() for t in Ws]
    mb = [t.clone() for t in bs]
    ring = [t.clone() for t in Ws]
    rb = [t.clone() for t in bs]
    act = [torch.empty(B, w, device="cuda") for _ in range(L - 1)]
    tmp = [torch.empty(B, w, device="cuda") for _ in range(2)]
    dzl = torch.empty(B, w, device="cuda")
    losses = []
    for s in range(steps):
        loss = torch.zeros(1, device="cuda")
        x = Xs[s]
        for l in range(L):
            if l < L - 1:
                nat.gemm(x, False, ring[l], False, B, w, w, kind=nat.EPI_STORE, out=act[l], bias=rb[l], relu=True)
                x = act[l]
            else:
                nat.gemm(x, False, ring[l], False, B, w, w, kind=nat.EPI_LOSS, out=dzl, bias=rb[l], target=Ts[s],
                         scale=1.0 / B, loss=loss)
        dz = dzl
        for l in range(L - 1, -1, -1):
            X = Xs[s] if l == 0 else act[l - 1]
            out = None
            if l > 0:
                out = tmp[l & 1]
                nat.gemm(dz, False, ring[l], True, B, w, w, kind=nat.EPI_MASK, out=out, mask=X)
            nat.gemm(dz, True, X, True, w, w, B, kind=nat.EPI_SGD, out=ring[l], master=mW[l], lr=lr)
            nat.bias_sgd(dz, B, w, mb[l], rb[l], lr)
            dz = out
        torch.cuda.synchronize()
        losses.append(float(loss))
    for s in range(steps):
        print(s, ref_losses[s], losses[s], abs(losses[s] - ref_losses[s]) / ref_losses[s])
    for l in range(L):
        d_ref = P[l] - Ws[l]
        print("layer", l, float((mW[l] - Ws[l] - d_ref).norm() / d_ref.norm()))


if __name__ == "__main__":
    kw = {k: (float(v) if "." in v or "e" in v else int(v)) for k, v in (a.split("=") for a in sys.argv[1:])}
    main(**kw)
