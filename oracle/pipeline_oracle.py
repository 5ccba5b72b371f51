"""CPU oracle for the pipeline-training hot path (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module, and only as the checker or the timed CPU
baseline; the product path (paper_1806_03377_b200) never calls it.

It restates, in numpy, the reference's numeric semantics of delayed SGD under
pipelining (pipesim/semantics.py):

* ``closed_form_version`` - the version each pass reads at a straight pipeline:
  stash max(0, mb - cap_s) for both passes (cap_s = n - s at NOAM; the
  simulator's staleness equation simulator.py:457-460 / semantics.py:211-217),
  vertical sync max(0, mb - cap_0) everywhere, naive forward like stash and
  naive backward mb - 1 (the latest commit at its start, simulator.py:243).
* ``toy_pipeline`` - the linear least-squares toy of semantics.py:39-116 run
  *as a pipeline*: stage s adds X_b[:, slice_s] @ w_s^(fwd version) to a running
  sum, the last stage forms the residual, the gradient flows back unchanged and
  dw_s = X_s^T r, applied to the latest weights (semantics.py:119-144, commit
  order of replay :169-191).  With fwd == bwd versions this equals
  ``equation_oracle`` (semantics.py:194-221) bit-for-bit up to summation order;
  tests pin it against the reference's own trajectories (tests/golden/toy_n*.npz).
* ``mlp_train`` - the same delayed-SGD rule for the MLP the device trains:
  forward with every stage's forward version, backward with each stage's
  backward version, update applied to the latest weights, minibatches committed
  in order 1..K.  ``emulate="bf16"`` rounds exactly where the device stores bf16
  (activations, dZ, weight-ring copies) while keeping fp32 master weights.

Parity status: schedule/ledger and the toy trajectories are pinned to the
reference's golden vectors; the MLP rule has no reference golden vector (the
reference has no MLP) and is pinned through ``toy_pipeline`` sharing its
version/commit logic.
"""

from __future__ import annotations

import numpy as np


# ---------------------------------------------------------------- versions (straight pipelines)
def caps_straight(n: int, max_inflight: int | None = None) -> list[int]:
    """cap_s = n - s, clipped by max_inflight (schedule.py:51-70 with replication 1)."""
    return [max(1, min(n - s, max_inflight) if max_inflight else n - s) for s in range(n)]


def closed_form_version(mode: str, n: int, s: int, mb: int, direction: str, max_inflight: int | None = None) -> int:
    caps = caps_straight(n, max_inflight)
    if mode == "vertical_sync":
        return max(0, mb - caps[0])
    if mode == "naive_pipeline" and direction == "backward":
        return mb - 1
    return max(0, mb - caps[s])


def closed_form_ledger(mode: str, n: int, K: int, max_inflight: int | None = None) -> dict:
    return {(s, mb, d): closed_form_version(mode, n, s, mb, d, max_inflight)
            for s in range(n) for mb in range(1, K + 1) for d in ("forward", "backward")}


# ---------------------------------------------------------------- linear toy pipeline
def toy_pipeline(design, targets, params, lr, block_size, versions, steps):
    """Trajectory (steps+1, n*p) of the toy model executed stage by stage.

    versions(s, mb, direction) -> int.  params: (n, p) initial blocks.
    """
    n, p = params.shape
    n_blocks = design.shape[0] // block_size
    archives = [[params[s].copy()] for s in range(n)]
    for mb in range(1, steps + 1):
        b = (mb - 1) % n_blocks
        xb = design[b * block_size:(b + 1) * block_size]
        yb = targets[b * block_size:(b + 1) * block_size]
        fv = [versions(s, mb, "forward") for s in range(n)]
        bv = [versions(s, mb, "backward") for s in range(n)]
        # forward: running sum of per-stage contributions
        run = np.zeros(block_size)
        for s in range(n):
            run = run + xb[:, s * p:(s + 1) * p] @ archives[s][fv[s]]
        resid = run - yb
        new = []
        for s in range(n):
            r = resid
            if bv[s] != fv[s]:  # own block re-read at the backward version (semantics.py:138-142)
                xs = xb[:, s * p:(s + 1) * p]
                r = resid + xs @ (archives[s][bv[s]] - archives[s][fv[s]])
            grad = xb[:, s * p:(s + 1) * p].T @ r
            new.append(archives[s][-1] - lr * grad)
        for s in range(n):
            archives[s].append(new[s])
    return np.stack([np.concatenate([archives[s][t] for s in range(n)]) for t in range(steps + 1)])


# ---------------------------------------------------------------- MLP
def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round to bfloat16 (nearest-even) and return as float64."""
    f = np.asarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def _fp32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def mlp_train(params, X, T, lr, stage_bounds, versions, K, emulate: str | None = None, dtype=np.float64,
              prune: bool = False, reps=None):
    """Delayed-SGD training of a ReLU MLP split into stages.

    params: list of (W [out,in], b [out]) per global layer; X: [n_blocks,B,d0]; T: [n_blocks,B,dL]
    stage_bounds: [(first, last)] 1-based layer ranges; versions(s, mb, dir) -> int.
    dtype: arithmetic type (float64 for parity, float32 for the timed CPU baseline).
    prune: drop weight versions no later minibatch reads (bounded memory for big models).
    reps: per-stage replication.  A stage replicated R ways follows the round rule of DESIGN.md §5:
      minibatches (k-1)R+1..kR form round k; their gradients (each at its own ledger versions) are
      summed and applied once to the latest weights, committing version kR.
    Returns (losses[K], final params list).  Loss per minibatch = 1/(2B) sum (Z - T)^2.
    """
    reps = list(reps) if reps is not None else [1] * len(stage_bounds)
    q = bf16_round if emulate == "bf16" else (lambda a: a)
    master = _fp32 if emulate == "bf16" else (lambda a: a)
    n = len(stage_bounds)
    L = len(params)
    layer_stage = {}
    for s, (a, b) in enumerate(stage_bounds):
        for l in range(a, b + 1):
            layer_stage[l - 1] = s
    # archives[s][v] = list of (W, b) for the stage's layers at version v (master precision)
    archives = [{0: [(master(np.asarray(params[l - 1][0], dtype=dtype)), master(np.asarray(params[l - 1][1], dtype=dtype)))
                     for l in range(a, b + 1)]}
                for (a, b) in stage_bounds]
    latest_v = [0] * n
    last_reader = [dict() for _ in range(n)]
    if prune:
        for mb in range(1, K + 1):
            for s in range(n):
                for d in ("forward", "backward"):
                    v = versions(s, mb, d)
                    last_reader[s][v] = max(last_reader[s].get(v, 0), mb)
    first = [a - 1 for a, _ in stage_bounds]
    n_blocks = X.shape[0]
    losses = []
    round_acc: dict = {}
    for mb in range(1, K + 1):
        blk = (mb - 1) % n_blocks
        x, t = np.asarray(X[blk], dtype=dtype), np.asarray(T[blk], dtype=dtype)
        B = x.shape[0]
        fv = [versions(s, mb, "forward") for s in range(n)]
        bv = [versions(s, mb, "backward") for s in range(n)]
        h = q(x)
        inputs = []
        z = None
        for l in range(L):
            s = layer_stage[l]
            W, b = archives[s][fv[s]][l - first[s]]
            inputs.append(h)
            z = h @ q(W).T + b
            if l < L - 1:
                h = q(np.maximum(z, 0.0))
        d = z - t
        losses.append(0.5 / B * float(np.sum(d * d)))
        dz = q(d / B)
        grads = [None] * L
        for l in range(L - 1, -1, -1):
            s = layer_stage[l]
            Xl = inputs[l]
            grads[l] = (dz.T @ Xl, dz.sum(axis=0))
            if l > 0:
                Wb, _ = archives[s][bv[s]][l - first[s]]
                dz = q((dz @ q(Wb)) * (Xl > 0))
        for s, (a, b) in enumerate(stage_bounds):
            R = reps[s]
            if R > 1:  # accumulate this minibatch's gradient into its round
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
            new = []
            for i in range(b - a + 1):
                W, bias = latest[i]
                gW, gb = step[i]
                new.append((master(W - lr * gW), master(bias - lr * gb)))
            archives[s][mb] = new
            latest_v[s] = mb
            if prune:
                for v in [v for v in archives[s] if v != mb and last_reader[s].get(v, 0) <= mb]:
                    del archives[s][v]
    final = []
    for s in range(n):
        final.extend(archives[s][latest_v[s]])
    return np.array(losses), final


def mlp_train_torch(params, X, T, lr, stage_bounds, versions, K, emulate: str | None = "bf16", device=None,
                    prune: bool = True, dtype=None, ksplit: int = 1, bias_grad_scale: float = 1.0):
    """``mlp_train``'s rule with torch fp32 arithmetic on ``device`` (the checker of full-size
    configurations, e.g. the 8 x 2-layer MLP-8192 at minibatch 2048, which numpy cannot run in
    seconds).  Same forward / backward versions, bf16 rounding points (fp32 -> bf16 nearest-even,
    as ``bf16_round``), fp32 master update onto the latest weights, in-order commits.  TF32 must be
    off (torch's default for matmul); straight pipelines only.

    params: [(W [out,in], b [out])] torch or numpy; X [n_blocks,B,d0]; T [n_blocks,B,dL].
    dtype: arithmetic type (default torch.float32; torch.float64 gives the exact-arithmetic reference
    against which an fp32 run's own rounding drift can be measured).
    ksplit: every product is summed over ``ksplit`` contiguous K chunks (a different fp32 summation
    order: the spread of such variants is the rounding-noise floor of fp32-accumulating GEMMs).
    bias_grad_scale: fault injection for the checker's own sensitivity test (1.0 = the rule).
    Returns (losses[K] numpy, final [(W, b)] torch tensors on ``device``).
    """
    import torch

    def mm(a, b):
        if ksplit <= 1:
            return a @ b
        kk = a.shape[1]
        step = (kk + ksplit - 1) // ksplit
        out = a[:, :step] @ b[:step]
        for k0 in range(step, kk, step):
            out = out + a[:, k0:k0 + step] @ b[k0:k0 + step]
        return out

    dtype = dtype or torch.float32

    def t32(a):
        return (a if isinstance(a, torch.Tensor) else torch.from_numpy(np.asarray(a))).to(device=device, dtype=dtype)

    # bf16 storage: round through fp32 (nearest-even); fp32 master weights
    q = (lambda a: a.float().bfloat16().to(dtype)) if emulate == "bf16" else (lambda a: a)
    mst = (lambda a: a.float().to(dtype)) if emulate == "bf16" else (lambda a: a)
    n = len(stage_bounds)
    L = len(params)
    layer_stage = {l - 1: s for s, (a, b) in enumerate(stage_bounds) for l in range(a, b + 1)}
    first = [a - 1 for a, _ in stage_bounds]
    archives = [{0: [(t32(params[l - 1][0]).clone(), t32(params[l - 1][1]).clone()) for l in range(a, b + 1)]}
                for (a, b) in stage_bounds]
    last_reader = [dict() for _ in range(n)]
    for mb in range(1, K + 1):
        for s in range(n):
            for d in ("forward", "backward"):
                v = versions(s, mb, d)
                last_reader[s][v] = max(last_reader[s].get(v, 0), mb)
    latest_v = [0] * n
    losses = []
    with torch.no_grad():
        for mb in range(1, K + 1):
            blk = (mb - 1) % X.shape[0]
            x, t = t32(X[blk]), t32(T[blk])
            B = x.shape[0]
            fv = [versions(s, mb, "forward") for s in range(n)]
            bv = [versions(s, mb, "backward") for s in range(n)]
            h = q(x)
            inputs = []
            z = None
            for l in range(L):
                s = layer_stage[l]
                W, b = archives[s][fv[s]][l - first[s]]
                inputs.append(h)
                z = mm(h, q(W).T) + b
                if l < L - 1:
                    h = q(torch.relu(z))
            d = z - t
            losses.append(0.5 / B * float((d.double() * d.double()).sum()))
            dz = q(d / B)
            grads = [None] * L
            for l in range(L - 1, -1, -1):
                s = layer_stage[l]
                Xl = inputs[l]
                grads[l] = (mm(dz.T, Xl), dz.sum(0) * bias_grad_scale)
                if l > 0:
                    Wb, _ = archives[s][bv[s]][l - first[s]]
                    dz = q(mm(dz, q(Wb)) * (Xl > 0))
            inputs = None
            for s, (a, b) in enumerate(stage_bounds):
                latest = archives[s][latest_v[s]]
                archives[s][mb] = [(mst(W - lr * grads[l][0]), mst(bias - lr * grads[l][1]))
                                   for (W, bias), l in zip(latest, range(a - 1, b))]
                latest_v[s] = mb
                if prune:
                    for v in [v for v in archives[s] if v != mb and last_reader[s].get(v, 0) <= mb]:
                        del archives[s][v]
            grads = None
    final = []
    for s in range(n):
        final.extend(archives[s][latest_v[s]])
    return np.array(losses), final
