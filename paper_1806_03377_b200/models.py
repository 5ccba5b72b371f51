"""Model specs the executor can run, their synthetic data and their layer profiles.

The reference models a network only as a chain of ``LayerProfile`` rows
(profiles.py:24-89) and its numerics only as the linear toy of
semantics.py:39-116.  The B200 executor runs real layers; profile layer l
(1-based) is ``Linear(widths[l-1] -> widths[l])`` followed by ReLU for every
layer but the last, and the loss is the mean-over-batch squared error
L = 1/(2B) * sum_b ||Z_b - T_b||^2 (the paper averages over the minibatch,
PAPER.md:623-624; the toy's 0.5*||r||^2 sum is its B=1 case).

Synthetic data follows semantics.py:76-80 and 93-116: one seeded
``numpy.random.default_rng(seed)`` (PCG64) stream, ``n_blocks`` input/target
blocks, minibatch m uses block (m-1) % n_blocks.  Weights ~ N(0, 2/d_in)
(He), biases ~ N(0, 0.01^2), inputs and targets ~ N(0, 1).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ValidationError
from .profiles import HardwareSpec, LayerProfile, ModelProfile, build_context

DTYPES = ("fp32", "bf16")


@dataclass(frozen=True)
class MLPSpec:
    widths: tuple[int, ...]  # d_0 .. d_L
    batch: int = 32
    dtype: str = "fp32"
    lr: float = 1e-3
    n_blocks: int = 8
    seed: int = 0

    def __post_init__(self):
        object.__setattr__(self, "widths", tuple(int(w) for w in self.widths))
        if len(self.widths) < 2:
            raise ValidationError("an MLP needs at least one layer (two widths)")
        if any(w < 1 for w in self.widths) or self.batch < 1 or self.n_blocks < 1:
            raise ValidationError("widths, batch and n_blocks must be positive")
        if self.dtype not in DTYPES:
            raise ValidationError(f"dtype must be one of {DTYPES}, got {self.dtype!r}")
        if self.lr < 0:
            raise ValidationError("lr must be >= 0")
        if self.dtype == "bf16" and any(w % 8 for w in self.widths):
            raise ValidationError("bf16 layers need widths that are multiples of 8 (16-byte TMA rows)")

    @property
    def num_layers(self) -> int:
        return len(self.widths) - 1

    @property
    def bytes_per_elem(self) -> int:
        return 4 if self.dtype == "fp32" else 2

    def flops_per_sample(self) -> float:
        """Algorithmic fwd+bwd FLOPs per sample: 6 * sum(d_in*d_out) minus the unneeded first dgrad."""
        macs = [a * b for a, b in zip(self.widths[:-1], self.widths[1:])]
        return 6.0 * sum(macs) - 2.0 * macs[0]


def mlp(width: int, layers: int, **kw) -> MLPSpec:
    return MLPSpec(widths=(width,) * (layers + 1), **kw)


def init_params(spec: MLPSpec) -> list[tuple[np.ndarray, np.ndarray]]:
    """Initial (W [out,in], b [out]) per layer, fp64, from the spec's seeded stream."""
    rng = np.random.default_rng(spec.seed)
    out = []
    for din, dout in zip(spec.widths[:-1], spec.widths[1:]):
        W = rng.normal(0.0, np.sqrt(2.0 / din), size=(dout, din))
        b = rng.normal(0.0, 0.01, size=dout)
        out.append((W, b))
    return out


def make_data(spec: MLPSpec) -> tuple[np.ndarray, np.ndarray]:
    """(X [n_blocks, B, d_0], T [n_blocks, B, d_L]) fp64; drawn after the parameters."""
    rng = np.random.default_rng([spec.seed, 1])
    X = rng.normal(0.0, 1.0, size=(spec.n_blocks, spec.batch, spec.widths[0]))
    T = rng.normal(0.0, 1.0, size=(spec.n_blocks, spec.batch, spec.widths[-1]))
    return X, T


def mlp_profile(spec: MLPSpec, tflops: float = 1000.0) -> ModelProfile:
    """Analytic per-layer profile (times from FLOPs at ``tflops``) for planning / prediction."""
    layers = []
    for l, (din, dout) in enumerate(zip(spec.widths[:-1], spec.widths[1:]), start=1):
        f = 2.0 * spec.batch * din * dout / (tflops * 1e12)
        layers.append(LayerProfile(l, f"linear{l}", f, 2.0 * f, spec.batch * dout, din * dout + dout))
    return ModelProfile(layers=tuple(layers), minibatch_size=spec.batch)


def mlp_context(spec: MLPSpec, machines: int = 1, bandwidth: float = 770e9, tflops: float = 1000.0):
    """CostContext for an MLP spec (bandwidth default: measured B200 NVLink peer copy)."""
    return build_context(mlp_profile(spec, tflops), HardwareSpec(machines, bandwidth, spec.bytes_per_elem))
