"""CPU oracle for GPT-2-style transformer pipelines (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this module, and only
as the checker or the timed CPU baseline; the product path never calls it.

``gpt_train`` applies the reference's delayed-SGD rule (pipesim/semantics.py:119-144: each
stage's forward/backward at its ledger version, the update applied to the latest weights,
minibatches committed in order as in replay :169-191; forward version == backward version, i.e.
weight stashing / vertical sync) to the model of ``paper_1806_03377_b200.models.GPTSpec``:
token + position embedding, pre-LN blocks (causal softmax attention over 64-wide heads,
tanh-GELU MLP), final LayerNorm, untied LM head, next-token softmax cross-entropy averaged over
all tokens (padded vocabulary columns excluded).  Arithmetic is torch CPU float64 autograd; with
``emulate="bf16"`` values are rounded to bf16 exactly where the device stores them (embedding
output, LN outputs, qkv, attention output, residual stream, FC1 pre-activation and GELU output,
weight-ring copies) and so are the gradients the device stores in bf16 (the same tensors'
gradients, and dlogits); the logits themselves stay fp32 on the device.  Attention internals
(the bf16 P tile before P.V) are not emulated; the tolerance in the tests covers them.

Parameter layout = the device's flat per-layer buffers (models.py GPTSpec / include/pd_b200.h
PD_LAYER_*).  Parity status: no reference golden vector exists for a transformer (the reference
has no tensors); the version/commit rule is the one pinned by toy_pipeline against the
reference's trajectories (tests/golden/toy_n*.npz).
"""

from __future__ import annotations

import numpy as np
import torch

F = torch.nn.functional


def _bf16(x: torch.Tensor) -> torch.Tensor:
    return x.float().bfloat16().to(x.dtype)


class _Q(torch.autograd.Function):
    """Round the value and its incoming gradient to bf16 (a bf16 tensor the device stores, whose
    gradient it also stores in bf16)."""

    @staticmethod
    def forward(ctx, x):
        return _bf16(x)

    @staticmethod
    def backward(ctx, g):
        return _bf16(g)


class _QF(torch.autograd.Function):
    """Round the value only (its gradient is consumed inside a fused epilogue)."""

    @staticmethod
    def forward(ctx, x):
        return _bf16(x)

    @staticmethod
    def backward(ctx, g):
        return g


class _QG(torch.autograd.Function):
    """Round the gradient only (fp32 logits, bf16 dlogits)."""

    @staticmethod
    def forward(ctx, x):
        return x.clone()

    @staticmethod
    def backward(ctx, g):
        return _bf16(g)


def _ident(x):
    return x


def _forward_loss(spec, weights, tok, lab, emulate):
    """Mean next-token CE of one minibatch; weights: per layer (W flat leaf, b leaf)."""
    Q = _Q.apply if emulate else _ident
    QF = _QF.apply if emulate else _ident
    QG = _QG.apply if emulate else _ident
    B, S = tok.shape
    d, f, H, Vp = spec.d, spec.ffn, spec.heads, spec.vocab_pad
    (We, _), blocks, (Wh, bh) = weights[0], weights[1:-1], weights[-1]
    We_q = QF(We)
    wte, wpe = We_q[:Vp], We_q[Vp:Vp + S]
    x = Q(wte[tok] + wpe[torch.arange(S, device=tok.device)].unsqueeze(0))  # [B, S, d]
    causal = torch.triu(torch.ones(S, S, dtype=torch.bool, device=tok.device), diagonal=1)
    for W, b in blocks:
        Wq = QF(W).reshape(-1)
        Wqkv = Wq[: 3 * d * d].view(3 * d, d)
        Wo = Wq[3 * d * d: 4 * d * d].view(d, d)
        W1 = Wq[4 * d * d: 4 * d * d + f * d].view(f, d)
        W2 = Wq[4 * d * d + f * d:].view(d, f)
        bqkv, bo, b1, b2 = b[: 3 * d], b[3 * d: 4 * d], b[4 * d: 4 * d + f], b[4 * d + f: 5 * d + f]
        g1, be1 = b[5 * d + f: 6 * d + f], b[6 * d + f: 7 * d + f]
        g2, be2 = b[7 * d + f: 8 * d + f], b[8 * d + f: 9 * d + f]
        h1 = Q(F.layer_norm(x, (d,), g1, be1, eps=1e-5))
        qkv = Q(h1 @ Wqkv.T + bqkv)
        q, k, v = qkv.split(d, dim=-1)
        q = q.view(B, S, H, 64).transpose(1, 2)
        k = k.view(B, S, H, 64).transpose(1, 2)
        v = v.view(B, S, H, 64).transpose(1, 2)
        att = (q @ k.transpose(-1, -2)) / 8.0
        att = att.masked_fill(causal, float("-inf")).softmax(-1)
        a = Q((att @ v).transpose(1, 2).reshape(B, S, d))
        x2 = Q(x + a @ Wo.T + bo)
        h2 = Q(F.layer_norm(x2, (d,), g2, be2, eps=1e-5))
        z = Q(h2 @ W1.T + b1)
        u = QF(F.gelu(z, approximate="tanh"))
        x = Q(x2 + u @ W2.T + b2)
    h = Q(F.layer_norm(x, (d,), bh[:d], bh[d:], eps=1e-5))
    logits = QG(h @ QF(Wh).T)[..., : spec.vocab]
    if emulate:
        logits = _QFP32.apply(logits)
    return F.cross_entropy(logits.reshape(B * S, -1), lab.reshape(-1).long())


class _QFP32(torch.autograd.Function):
    """fp32 logits (the device's GEMM output precision)."""

    @staticmethod
    def forward(ctx, x):
        return x.float().to(x.dtype)

    @staticmethod
    def backward(ctx, g):
        return g


def _as_t(a, dtype, device):
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=dtype).clone()
    return torch.from_numpy(np.asarray(a)).to(device=device, dtype=dtype).clone()


def _as_i(a, device):
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=torch.int64)
    return torch.from_numpy(np.asarray(a, np.int64)).to(device)


def gpt_train(spec, params, X, labels, lr, stage_bounds, versions, K, emulate: str | None = "bf16",
              dtype=torch.float64, device=None):
    """Delayed-SGD pipeline training of a GPTSpec model (see module docstring).

    params: [(W, b)] per profile layer (device layout), numpy or torch; X, labels: [n_blocks, B, S] ints.
    dtype: arithmetic type (float64 for parity; float32 for the timed CPU baseline, or on a GPU for
    full-size checks with TF32 off).  device: torch device of the arithmetic (default CPU).
    Returns (losses[K], final params list of (W, b)): numpy fp64 on the CPU, torch tensors on a device.
    """
    emul = emulate == "bf16"
    master = (lambda a: a.float().to(a.dtype)) if emul else (lambda a: a)
    n = len(stage_bounds)
    layer_stage = {}
    for s, (a, b) in enumerate(stage_bounds):
        for l in range(a, b + 1):
            layer_stage[l - 1] = s
    first = [a - 1 for a, _ in stage_bounds]
    archives = [{0: [(master(_as_t(params[l - 1][0], dtype, device)), master(_as_t(params[l - 1][1], dtype, device)))
                     for l in range(a, b + 1)]} for (a, b) in stage_bounds]
    latest_v = [0] * n
    losses = []
    L = len(params)
    for mb in range(1, K + 1):
        blk = (mb - 1) % X.shape[0]
        tok = _as_i(X[blk], device)
        lab = _as_i(labels[blk], device)
        fv = [versions(s, mb, "forward") for s in range(n)]
        if fv != [versions(s, mb, "backward") for s in range(n)]:
            raise ValueError("gpt_train supports forward version == backward version only")
        leaves = []
        for l in range(L):
            s = layer_stage[l]
            W, b = archives[s][fv[s]][l - first[s]]
            leaves.append((W.clone().requires_grad_(True), b.clone().requires_grad_(True)))
        with torch.enable_grad():
            loss = _forward_loss(spec, leaves, tok, lab, emul)
            loss.backward()
        losses.append(float(loss.detach()))
        for s, (a, b) in enumerate(stage_bounds):
            latest = archives[s][latest_v[s]]
            new = []
            for i, l in enumerate(range(a - 1, b)):
                W, bias = latest[i]
                gW, gb = leaves[l][0].grad, leaves[l][1].grad
                gb = torch.zeros_like(bias) if gb is None else gb
                new.append((master(W - lr * gW), master(bias - lr * gb)))
            archives[s][mb] = new
            latest_v[s] = mb
    final = []
    for s in range(n):
        if device is not None:
            final.extend(archives[s][latest_v[s]])
        else:
            final.extend((W.double().numpy(), b.double().numpy()) for W, b in archives[s][latest_v[s]])
    return np.array(losses), final
