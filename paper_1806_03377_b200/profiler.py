"""B200 layer profiler: measured per-layer costs as a reference-format ``ModelProfile``.

PipeDream partitions on *measured* per-layer times (the reference reads
them from JSON, profiles.py:112-187).  This profiler times each MLP layer with the same
kernels the executor runs (CUDA events, after warm-up):
  fwd_time = forward GEMM with its fused bias+ReLU epilogue (or the loss epilogue on the
             last layer),
  bwd_time = dgrad (+ReLU mask) + wgrad with the fused SGD update + bias update,
and records activation_elems = B*d_out, param_elems = d_in*d_out + d_out.  The result
round-trips through ``save_profile`` into the reference's JSON format, so either package's
``solve`` can plan on it.
"""

from __future__ import annotations

import ctypes

from . import _native as nat
from .models import ConvNetSpec, GPTSpec, MLPSpec
from .profiles import LayerProfile, ModelProfile


def profile_mlp(spec: MLPSpec, repeats: int = 10, warmup: int = 3, device=None) -> ModelProfile:
    import torch

    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    dt = torch.float32 if spec.dtype == "fp32" else torch.bfloat16
    B = spec.batch
    layers = []
    L = spec.num_layers
    for l, (din, dout) in enumerate(zip(spec.widths[:-1], spec.widths[1:]), start=1):
        X = torch.randn(B, din, device=dev).to(dt)
        W = (torch.randn(dout, din, device=dev) * (2.0 / din) ** 0.5).to(dt)
        master = W.float()
        ring = torch.empty_like(W)
        bias = torch.zeros(dout, device=dev)
        bias_out = torch.empty_like(bias)
        Y = torch.empty(B, dout, device=dev, dtype=dt)
        dZ = torch.randn(B, dout, device=dev).to(dt)
        dX = torch.empty(B, din, device=dev, dtype=dt)
        target = torch.randn(B, dout, device=dev)
        loss = torch.zeros(1, device=dev)

        def fwd():
            if l < L:
                nat.gemm(X, False, W, False, B, dout, din, kind=nat.EPI_STORE, out=Y, bias=bias, relu=True)
            else:
                nat.gemm(X, False, W, False, B, dout, din, kind=nat.EPI_LOSS, out=Y, bias=bias, target=target,
                         scale=1.0 / B, loss=loss)

        def bwd():
            if l > 1:
                nat.gemm(dZ, False, W, True, B, din, dout, kind=nat.EPI_MASK, out=dX, mask=X)
            nat.gemm(dZ, True, X, True, dout, din, B, kind=nat.EPI_SGD, out=ring, master=master, lr=0.0)
            nat.bias_sgd(dZ, B, dout, bias, bias_out, 0.0)

        times = []
        for fn in (fwd, bwd):
            for _ in range(warmup):
                fn()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(dev)
            a.record()
            for _ in range(repeats):
                fn()
            b.record()
            torch.cuda.synchronize(dev)
            times.append(a.elapsed_time(b) / repeats * 1e-3)
        layers.append(LayerProfile(l, f"linear{l}_{din}x{dout}", times[0], times[1], B * dout, din * dout + dout))
    return ModelProfile(layers=tuple(layers), minibatch_size=B)


def _layer_names(spec) -> list[str]:
    if isinstance(spec, MLPSpec):
        return [f"linear{l}_{a}x{b}" for l, (a, b) in enumerate(zip(spec.widths[:-1], spec.widths[1:]), start=1)]
    names = []
    for l, g in enumerate(spec.geoms(), start=1):
        if g.kind == "conv":
            names.append(f"conv{l}_{g.h}x{g.w}x{g.c_in}-{g.c_out}" + ("_pool" if g.pool else ""))
        elif g.kind == "linear":
            names.append(f"fc{l}_{g.c_in}x{g.c_out}")
        else:
            names.append(f"{g.kind}{l}")
    return names


def profile_model(spec, minibatches: int = 12, steps: int = 2, device=None) -> ModelProfile:
    """Measured per-layer profile of any executor model (MLP, ConvNet, GPT) as a reference-format
    ``ModelProfile``: the whole model runs as ONE stage through the executor's own kernel chains
    (so conv pools, attention, LayerNorm, losses and the fused updates are all included) with
    per-layer CUDA events on the stage stream; fwd_time / bwd_time are the averages over
    ``steps`` runs of ``minibatches`` minibatches.  activation_elems = batch x the layer's output
    features (the message a stage boundary after this layer would carry), param_elems = its
    weights + biases.  Feed it to ``solve`` to partition on B200 measurements."""
    import torch

    from .executor import Executor
    from .ledger import SimConfig
    from .plans import Plan, Stage

    L = spec.num_layers
    plan = Plan(stages=(Stage(1, L, 1),), bottleneck_time=1.0, noam=1, machines_used=1)
    cfg = SimConfig(plan=plan, mode="weight_stashing", num_minibatches=max(11, minibatches))
    ex = Executor(cfg, model=spec, device=device)
    try:
        ex.set_serial(True)
        ex.set_graph(True)  # replayed as a CUDA graph: no host launch gaps inside the timed layers
        ex.step()  # warm-up (tensor maps, attributes, caches)
        torch.cuda.synchronize(ex.device)
        lib = nat.lib()
        cap = 2 * L * cfg.num_minibatches + 16  # stamps of one run (a replay rewrites the same slots)
        ts = torch.zeros(2 * cap, dtype=torch.int64, device=ex.device)
        nat.check(lib.pd_rt_layer_timing(ex._rt, ts.data_ptr(), cap), "pd_rt_layer_timing")
        for _ in range(steps + 1):  # the first run captures the graph (with the stamp kernels)
            ex.step()
        torch.cuda.synchronize(ex.device)
        buf = (ctypes.c_double * (2 * L))()
        nat.check(lib.pd_rt_layer_stats(ex._rt, 0, L, buf), "pd_rt_layer_stats")
        nat.check(lib.pd_rt_layer_timing(ex._rt, None, 0), "pd_rt_layer_timing")
    finally:
        ex.close()
    names = _layer_names(spec)
    if isinstance(spec, MLPSpec):
        outs = list(spec.widths[1:])
        params = [a * b + b for a, b in zip(spec.widths[:-1], spec.widths[1:])]
    else:
        geo = spec.geoms()
        outs = [g.out_features for g in geo]
        params = [g.w_numel + g.b_numel for g in geo]
    layers = tuple(LayerProfile(l + 1, names[l], buf[2 * l] * 1e-3, buf[2 * l + 1] * 1e-3, spec.batch * outs[l],
                                params[l]) for l in range(L))
    return ModelProfile(layers=layers, minibatch_size=spec.batch)
