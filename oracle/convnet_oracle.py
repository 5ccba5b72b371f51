"""CPU oracle for convolutional pipeline stages (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this module, and only
as the checker or the timed CPU baseline; the product path never calls it.

``convnet_train`` applies the delayed-SGD rule of the reference (pipesim/semantics.py:119-144:
every stage's forward at its forward version, its backward at its backward version, the update
applied to the *latest* weights; minibatches committed in order, replay :169-191) to a VGG-style
network: 3x3/pad-1 convolutions + ReLU (+ 2x2 max pool), Linear layers, softmax cross-entropy
(mean over the minibatch).  It is the same rule ``pipeline_oracle.mlp_train`` restates for the
MLP, whose version/commit logic is pinned to the reference's golden trajectories through
``toy_pipeline`` (tests/golden/toy_n*.npz); replicated stages follow the round rule of
DESIGN.md §5.  Arithmetic is torch CPU float64 with ``emulate="bf16"`` rounding exactly where
the device stores bf16 (images, activations, activation gradients, weight-ring copies) and fp32
master weights; the loss logits stay fp32 on the device, so they are not rounded here.

Max pool: window scan order (0,0),(0,1),(1,0),(1,1), the first maximum wins (the device rule).
Weights: conv layers are Wt [9*c_in (or 64 for the im2col'ed image layer), c_out] with row
(r*3+s)*c_in + c; Linear layers W [c_out, c_in]; NHWC activations, flattened in NHWC order.
Only weight stashing / vertical sync (forward version == backward version) are supported.
Parity status: no reference golden vector exists for a convolutional network (the reference has
no tensors); pinned through the shared version rule as above.
"""

from __future__ import annotations

import numpy as np
import torch


F = torch.nn.functional


def _q_t(x: torch.Tensor) -> torch.Tensor:
    """Round to bf16 through fp32 (nearest-even both times), as pipeline_oracle.bf16_round does."""
    return x.float().bfloat16().to(x.dtype)


def _as_t(a, dtype, device) -> torch.Tensor:
    """numpy array or torch tensor -> torch tensor of dtype on device (the oracle may run on a GPU
    as the checker of full-size configurations; its arithmetic is the same)."""
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=dtype)
    return torch.from_numpy(np.asarray(a, np.float64)).to(device=device, dtype=dtype)


def _f32_t(x: torch.Tensor) -> torch.Tensor:
    return x.float().to(x.dtype)


def _oihw(Wt: torch.Tensor, cin: int, cout: int) -> torch.Tensor:
    return Wt[: 9 * cin].reshape(3, 3, cin, cout).permute(3, 2, 0, 1)


def _pool_fwd(y: torch.Tensor):
    n, h, w, c = y.shape
    win = y.reshape(n, h // 2, 2, w // 2, 2, c).permute(0, 1, 3, 5, 2, 4).reshape(n, h // 2, w // 2, c, 4)
    v, _ = win.max(-1)
    arg = (win == v.unsqueeze(-1)).double().argmax(-1)  # first maximum in scan order
    return v, arg


def _pool_bwd(dz: torch.Tensor, arg: torch.Tensor):
    n, ho, wo, c = dz.shape
    out = torch.zeros(n, ho, wo, c, 4, dtype=dz.dtype, device=dz.device)
    out.scatter_(-1, arg.unsqueeze(-1), dz.unsqueeze(-1))
    return out.reshape(n, ho, wo, c, 2, 2).permute(0, 1, 4, 2, 5, 3).reshape(n, 2 * ho, 2 * wo, c)


def _forward(geoms, weights, x, q):
    """Returns (logits, per-layer saved (input, aux))."""
    saved = []
    h = q(x)
    B = x.shape[0]
    for g, (W, b) in zip(geoms, weights):
        if g.kind == "conv":
            xin = h.reshape(B, g.h, g.w, g.c_in)
            z = F.conv2d(xin.permute(0, 3, 1, 2), _oihw(q(W), g.c_in, g.c_out), b, padding=1).permute(0, 2, 3, 1)
            y = q(torch.relu(z))
            arg = None
            if g.pool:
                y, arg = _pool_fwd(y)
            saved.append((xin, arg))
            h = y.reshape(B, -1)
        else:
            xin = h.reshape(B, -1)
            z = xin @ q(W).T + b
            saved.append((xin, None))
            h = q(torch.relu(z)) if g.relu else z
    return h, saved


def _backward(geoms, weights, saved, dz, q):
    """Gradients [(dW, db)] per layer, dz = dL/d(logits) (already rounded)."""
    grads = [None] * len(geoms)
    for l in range(len(geoms) - 1, -1, -1):
        g = geoms[l]
        W, _ = weights[l]
        xin, arg = saved[l]
        B = xin.shape[0]
        if g.kind == "conv":
            d = dz.reshape(B, g.h // 2 if g.pool else g.h, g.w // 2 if g.pool else g.w, g.c_out)
            dy = _pool_bwd(d, arg) if g.pool else d
            dW = torch.nn.grad.conv2d_weight(xin.permute(0, 3, 1, 2), (g.c_out, g.c_in, 3, 3), dy.permute(0, 3, 1, 2),
                                             padding=1)
            gWt = torch.zeros(g.w_shape, dtype=dW.dtype, device=dW.device)
            gWt[: 9 * g.c_in] = dW.permute(2, 3, 1, 0).reshape(9 * g.c_in, g.c_out)
            grads[l] = (gWt, dy.reshape(-1, g.c_out).sum(0))
            if l > 0:
                dx = torch.nn.grad.conv2d_input((B, g.c_in, g.h, g.w), _oihw(q(W), g.c_in, g.c_out),
                                                dy.permute(0, 3, 1, 2), padding=1).permute(0, 2, 3, 1)
                dz = q(dx * (xin > 0)).reshape(B, -1)
        else:
            grads[l] = (dz.T @ xin, dz.sum(0))
            if l > 0:
                dz = q((dz @ q(W)) * (xin > 0))
    return grads


@torch.no_grad()
def convnet_train(geoms, params, X, labels, lr, stage_bounds, versions, K, emulate: str | None = "bf16", reps=None,
                  dtype=torch.float64, device=None):
    """Delayed-SGD pipeline training of a conv net (see module docstring).

    geoms: per-layer geometry objects (kind, h, w, c_in, c_out, pool, relu, w_shape);
    params: [(W, b)] per layer, numpy or torch; X [n_blocks, B, H, W, C]; labels [n_blocks, B].
    dtype: arithmetic type (float64 for parity; float32 for the timed CPU baseline, or on a GPU for
    full-size checks with TF32 off).  device: torch device of the arithmetic (default CPU).
    Returns (losses[K], final params list of (W, b)): numpy fp64 on the CPU, torch tensors on a device.
    """
    q = _q_t if emulate == "bf16" else (lambda a: a)
    master = _f32_t if emulate == "bf16" else (lambda a: a)
    n = len(stage_bounds)
    reps = list(reps) if reps is not None else [1] * n
    layer_stage = {}
    for s, (a, b) in enumerate(stage_bounds):
        for l in range(a, b + 1):
            layer_stage[l - 1] = s
    archives = [{0: [(master(_as_t(params[l - 1][0], dtype, device)), master(_as_t(params[l - 1][1], dtype, device)))
                     for l in range(a, b + 1)]}
                for (a, b) in stage_bounds]
    latest_v = [0] * n
    first = [a - 1 for a, _ in stage_bounds]
    losses, round_acc = [], {}
    for mb in range(1, K + 1):
        blk = (mb - 1) % X.shape[0]
        x = _as_t(X[blk], dtype, device)
        y = labels[blk].to(device=device, dtype=torch.int64) if isinstance(labels, torch.Tensor) else \
            torch.from_numpy(np.asarray(labels[blk], np.int64)).to(device)
        B = x.shape[0]
        fv = [versions(s, mb, "forward") for s in range(n)]
        bv = [versions(s, mb, "backward") for s in range(n)]
        if fv != bv:
            raise ValueError("convnet_train supports forward version == backward version only")
        weights = [archives[layer_stage[l]][fv[layer_stage[l]]][l - first[layer_stage[l]]] for l in range(len(geoms))]
        logits, saved = _forward(geoms, weights, x, q)
        logits = logits.float().to(logits.dtype) if emulate == "bf16" else logits  # fp32 logits on the device
        lse = torch.logsumexp(logits, dim=1)
        rows = torch.arange(B, device=logits.device)
        losses.append(float((lse - logits[rows, y]).mean()))
        p = torch.softmax(logits, dim=1)
        p[rows, y] -= 1.0
        dz = q(p / B)
        grads = _backward(geoms, weights, saved, dz, q)
        for s, (a, b) in enumerate(stage_bounds):
            R = reps[s]
            if R > 1:
                acc = round_acc.setdefault(s, [None] * (b - a + 1))
                for i, l in enumerate(range(a - 1, b)):
                    gW, gb = grads[l]
                    acc[i] = (gW, gb) if acc[i] is None else (acc[i][0] + gW, acc[i][1] + gb)
                if mb % R:
                    continue
                step = round_acc.pop(s)
            else:
                step = [grads[l] for l in range(a - 1, b)]
            latest = archives[s][latest_v[s]]
            archives[s][mb] = [(master(W - lr * gW), master(bias - lr * gb))
                               for (W, bias), (gW, gb) in zip(latest, step)]
            latest_v[s] = mb
    final = []
    for s in range(n):
        if device is not None:
            final.extend(archives[s][latest_v[s]])
        else:
            final.extend((W.double().numpy(), b.double().numpy()) for W, b in archives[s][latest_v[s]])
    return np.array(losses), final
