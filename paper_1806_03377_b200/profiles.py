"""Layer profiles, hardware description and the analytic cost model.

These are inputs of the hot path, not part of it: ``run()`` receives a
``CostContext`` exactly like the reference's ``pipesim.run(cfg, ctx)``.
Field names, units (seconds, element counts, bytes/s) and formulas follow
pipesim/profiles.py:24-106 and pipesim/costmodel.py:27-138 so a context built
by either package means the same thing.  The executor only uses the context
for validation (plan/profile layer count, simulator.py:153-156) and for the
"predicted" columns printed beside measured numbers.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path
from typing import TYPE_CHECKING

from .errors import ProfileFormatError, ValidationError

if TYPE_CHECKING:  # pragma: no cover
    from .plans import Plan

DEFAULT_BYTES_PER_ELEM = 4


@dataclass(frozen=True)
class LayerProfile:
    """Per-minibatch cost of one layer (profiles.py:24-56): times in s, sizes in elements."""

    layer_id: int
    name: str
    fwd_time: float
    bwd_time: float
    activation_elems: int
    param_elems: int

    def __post_init__(self):
        where = f"layer {self.layer_id} ({self.name})"
        checks = (
            (self.fwd_time >= 0, "fwd_time must be >= 0"),
            (self.bwd_time >= 0, "bwd_time must be >= 0"),
            (self.fwd_time + self.bwd_time > 0, "fwd_time + bwd_time must be > 0"),
            (self.activation_elems >= 0, "activation_elems must be >= 0"),
            (self.param_elems >= 0, "param_elems must be >= 0"),
        )
        for ok, msg in checks:
            if not ok:
                raise ValidationError(f"{where}: {msg}")

    @property
    def total_time(self) -> float:
        return self.fwd_time + self.bwd_time


@dataclass(frozen=True)
class ModelProfile:
    layers: tuple[LayerProfile, ...]
    minibatch_size: int = 32

    def __post_init__(self):
        object.__setattr__(self, "layers", tuple(self.layers))
        if not self.layers:
            raise ValidationError("profile must contain at least one layer")
        for want, layer in enumerate(self.layers, start=1):
            if layer.layer_id != want:
                raise ValidationError(
                    f"layer_id values must be exactly 1..N in order; position {want} has layer_id {layer.layer_id}"
                )
        if self.minibatch_size <= 0:
            raise ValidationError("minibatch_size must be > 0")

    @property
    def num_layers(self) -> int:
        return len(self.layers)

    @property
    def total_time(self) -> float:
        return sum(layer.total_time for layer in self.layers)

    @property
    def total_param_elems(self) -> int:
        return sum(layer.param_elems for layer in self.layers)


@dataclass(frozen=True)
class HardwareSpec:
    num_machines: int
    bandwidth: float  # bytes/s of the inter-stage link
    bytes_per_elem: int = DEFAULT_BYTES_PER_ELEM

    def __post_init__(self):
        if self.num_machines < 1:
            raise ValidationError("num_machines must be >= 1")
        if self.bandwidth <= 0:
            raise ValidationError("bandwidth must be > 0")
        if self.bytes_per_elem <= 0:
            raise ValidationError("bytes_per_elem must be > 0")


def load_profile(path: str | Path) -> ModelProfile:
    """JSON ``{"minibatch_size", "layers": [{name, fwd_time, bwd_time, activation_elems, param_elems}]}``."""
    try:
        doc = json.loads(Path(path).read_text())
        layers = tuple(
            LayerProfile(
                i + 1, str(d["name"]), float(d["fwd_time"]), float(d["bwd_time"]),
                int(d["activation_elems"]), int(d["param_elems"]),
            )
            for i, d in enumerate(doc["layers"])
        )
        return ModelProfile(layers=layers, minibatch_size=int(doc.get("minibatch_size", 32)))
    except (OSError, KeyError, TypeError, ValueError) as exc:
        if isinstance(exc, ValidationError):
            raise
        raise ProfileFormatError(f"{path}: {exc}") from exc


def save_profile(profile: ModelProfile, path: str | Path) -> None:
    doc = {
        "minibatch_size": profile.minibatch_size,
        "layers": [
            {
                "name": l.name, "fwd_time": l.fwd_time, "bwd_time": l.bwd_time,
                "activation_elems": l.activation_elems, "param_elems": l.param_elems,
            }
            for l in profile.layers
        ],
    }
    Path(path).write_text(json.dumps(doc, indent=2))


# ------------------------------------------------------------------ cost model (costmodel.py)


@dataclass(frozen=True)
class CostContext:
    """Profile + hardware + prefix sums; prefix_T[k] = fwd+bwd time of layers 1..k."""

    profile: ModelProfile
    hw: HardwareSpec
    prefix_T: tuple[float, ...]
    prefix_W_bytes: tuple[float, ...]

    @property
    def num_layers(self) -> int:
        return self.profile.num_layers


def build_context(profile: ModelProfile, hw: HardwareSpec) -> CostContext:
    t, w = [0.0], [0.0]
    for layer in profile.layers:
        t.append(t[-1] + layer.total_time)
        w.append(w[-1] + float(layer.param_elems * hw.bytes_per_elem))
    return CostContext(profile=profile, hw=hw, prefix_T=tuple(t), prefix_W_bytes=tuple(w))


def _span(ctx, i: int, j: int, m: int) -> None:
    if not 1 <= i <= j <= ctx.num_layers:
        raise ValidationError(f"layer range {i}..{j} invalid for N={ctx.num_layers}")
    if m < 1:
        raise ValidationError(f"replication must be >= 1, got {m}")


def compute_time(ctx, i: int, j: int) -> float:
    _span(ctx, i, j, 1)
    return ctx.prefix_T[j] - ctx.prefix_T[i - 1]


def comm_time_activations(ctx, l: int) -> float:
    """Seconds to move layer l's output across boundary l -> l+1 (costmodel.py:68-79)."""
    if not 1 <= l <= ctx.num_layers - 1:
        raise ValidationError(f"boundary index must satisfy 1 <= l <= N-1 (N={ctx.num_layers}), got {l}")
    return ctx.profile.layers[l - 1].activation_elems * ctx.hw.bytes_per_elem / ctx.hw.bandwidth


def weight_sync_time(ctx, i: int, j: int, m: int) -> float:
    """(m-1)/m * stage weight bytes / bandwidth; 0 for m == 1 (costmodel.py:82-92)."""
    _span(ctx, i, j, m)
    if m == 1:
        return 0.0
    return (m - 1) / m * (ctx.prefix_W_bytes[j] - ctx.prefix_W_bytes[i - 1]) / ctx.hw.bandwidth


def stage_time(ctx, i: int, j: int, m: int) -> float:
    """max(compute, sync) / m (costmodel.py:95-103)."""
    _span(ctx, i, j, m)
    return max(compute_time(ctx, i, j), weight_sync_time(ctx, i, j, m)) / m


def comm_volume_bsp(ctx, m: int) -> float:
    if m < 1:
        raise ValidationError(f"machine count must be >= 1, got {m}")
    return (m - 1) * ctx.prefix_W_bytes[-1]


def comm_volume_pp(ctx, plan: "Plan") -> float:
    """Bytes per minibatch of a plan: 2*a*bpe per internal boundary + replicated-stage sync."""
    st = plan.stages
    if st[0].first_layer != 1 or st[-1].last_layer != ctx.num_layers:
        raise ValidationError(
            f"plan covers layers {st[0].first_layer}..{st[-1].last_layer}, profile has N={ctx.num_layers}"
        )
    total = 0.0
    for k, s in enumerate(st):
        if k + 1 < len(st):
            total += 2.0 * ctx.profile.layers[s.last_layer - 1].activation_elems * ctx.hw.bytes_per_elem
        if s.replication > 1:
            total += (s.replication - 1) * (ctx.prefix_W_bytes[s.last_layer] - ctx.prefix_W_bytes[s.first_layer - 1])
    return total
