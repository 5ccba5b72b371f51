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

from . import _native as nat
from .models import MLPSpec
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
