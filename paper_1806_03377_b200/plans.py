"""Plan / Stage types consumed by the executor (pipesim/partitioner.py:36-180).

A plan is the partitioner's output: contiguous layer ranges, each served by
``replication`` GPUs, plus NOAM (the number of minibatches the input stage keeps
in flight).  Objects from the reference package work too: everything here
reads only ``.stages[i].first_layer/last_layer/replication``, ``.noam`` and
``.machines_used``.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path

from .errors import ValidationError
from .profiles import comm_time_activations, stage_time


@dataclass(frozen=True)
class Stage:
    first_layer: int
    last_layer: int
    replication: int

    def __post_init__(self):
        if self.first_layer > self.last_layer:
            raise ValidationError(f"stage range {self.first_layer}..{self.last_layer} is empty")
        if self.replication < 1:
            raise ValidationError("stage replication must be >= 1")

    @property
    def num_layers(self) -> int:
        return self.last_layer - self.first_layer + 1


def noam_for(machines_used: int, input_replication: int) -> int:
    """ceil(machines / input-stage replication) (partitioner.py:127-130)."""
    return -(-machines_used // input_replication)


@dataclass(frozen=True)
class Plan:
    stages: tuple[Stage, ...]
    bottleneck_time: float
    noam: int
    machines_used: int

    def __post_init__(self):
        object.__setattr__(self, "stages", tuple(self.stages))
        if not self.stages:
            raise ValidationError("plan must contain at least one stage")
        if self.stages[0].first_layer != 1:
            raise ValidationError("plan must start at layer 1")
        for prev, nxt in zip(self.stages, self.stages[1:]):
            if nxt.first_layer != prev.last_layer + 1:
                raise ValidationError("plan stages must cover layers contiguously")
        if self.machines_used != sum(s.replication for s in self.stages):
            raise ValidationError("machines_used must equal the sum of replications")
        if self.noam != noam_for(self.machines_used, self.stages[0].replication):
            raise ValidationError("noam does not match ceil(machines / input replication)")

    @property
    def num_layers(self) -> int:
        return self.stages[-1].last_layer

    @property
    def num_stages(self) -> int:
        return len(self.stages)

    @property
    def config_string(self) -> str:
        return "-".join(str(s.replication) for s in self.stages)

    def to_dict(self) -> dict:
        return {
            "stages": [
                {"first_layer": s.first_layer, "last_layer": s.last_layer, "replication": s.replication}
                for s in self.stages
            ],
            "bottleneck_time": self.bottleneck_time,
            "noam": self.noam,
            "machines_used": self.machines_used,
        }


def noam(plan) -> int:
    return noam_for(plan.machines_used, plan.stages[0].replication)


def plan_from_dict(doc: dict) -> Plan:
    try:
        return Plan(
            stages=tuple(Stage(d["first_layer"], d["last_layer"], d["replication"]) for d in doc["stages"]),
            bottleneck_time=float(doc["bottleneck_time"]),
            noam=int(doc["noam"]),
            machines_used=int(doc["machines_used"]),
        )
    except (KeyError, TypeError) as exc:
        raise ValidationError(f"malformed plan document: {exc}") from exc


def load_plan(path: str | Path) -> Plan:
    return plan_from_dict(json.loads(Path(path).read_text()))


def parse_config(text: str, n_layers: int | None = None) -> list[int]:
    """'7-1' -> [7, 1] (partitioner.py:137-158)."""
    reps = []
    for part in text.strip().split("-"):
        try:
            value = int(part)
        except ValueError as exc:
            raise ValidationError(f"config {text!r}: {part!r} is not an integer") from exc
        if value < 1:
            raise ValidationError(f"config {text!r}: replication must be positive")
        reps.append(value)
    if n_layers is not None and len(reps) > n_layers:
        raise ValidationError(f"config {text!r} has {len(reps)} stages but the model has {n_layers} layers")
    return reps


def straight_plan(ctx, stage_bounds) -> Plan:
    """Replication-1 plan over explicit (first, last) layer ranges (partitioner.py:171-180)."""
    stages = tuple(Stage(a, b, 1) for a, b in stage_bounds)
    times = [stage_time(ctx, s.first_layer, s.last_layer, 1) for s in stages]
    links = [2.0 * comm_time_activations(ctx, s.last_layer) for s in stages[:-1]]
    return Plan(stages=stages, bottleneck_time=max(times + links), noam=len(stages), machines_used=len(stages))


def replicated_plan(ctx, stage_specs) -> Plan:
    """Plan from explicit ((first, last), replication) specs, e.g. VGG-16 7-1."""
    stages = tuple(Stage(a, b, r) for (a, b), r in stage_specs)
    times = [stage_time(ctx, s.first_layer, s.last_layer, s.replication) for s in stages]
    links = [2.0 * comm_time_activations(ctx, s.last_layer) for s in stages[:-1]]
    used = sum(s.replication for s in stages)
    return Plan(stages=stages, bottleneck_time=max(times + links), noam=noam_for(used, stages[0].replication),
                machines_used=used)


# ------------------------------------------------------------------ planner (partitioner.py:183-308)
TIME_TOL = 1e-12  # float ties in the DP are decided by structure, not evaluation order


def _better(a, b) -> bool:
    """Candidate a = (time, n_stages, split, split_m) strictly preferred over b (or b is None)."""
    if b is None:
        return True
    if a[0] < b[0] - TIME_TOL:
        return True
    if a[0] > b[0] + TIME_TOL:
        return False
    return a[1:] < b[1:]  # fewer stages, then earlier last split, then smaller final replication


def solve(ctx, machines: int | None = None, *, force_all_machines: bool = False,
          max_replication: int | None = None, stats: dict | None = None) -> Plan:
    """Bottleneck-minimising contiguous partition with per-stage replication (PipeDream §3.1).

    best[j][m] is the best pipeline over layers 1..j on exactly m machines: either one stage
    replicated m ways, or best[i][m - m'] followed by a stage over i+1..j on m' machines, with the
    boundary i paying 2*C_i.  Same tie rules and outputs as the reference's ``solve``, so a plan
    computed from a B200-measured profile (profiler.py) feeds ``run`` directly.
    """
    n = ctx.num_layers
    budget = ctx.hw.num_machines if machines is None else machines
    if budget < 1:
        raise ValidationError("machine budget must be >= 1")
    cap = budget if max_replication is None else max_replication
    if cap < 1:
        raise ValidationError("max_replication must be >= 1")
    link = [0.0] + [2.0 * comm_time_activations(ctx, i) for i in range(1, n)]
    best = [[None] * (budget + 1) for _ in range(n + 1)]
    evals = 0
    for j in range(1, n + 1):
        for m in range(1, budget + 1):
            cell = (stage_time(ctx, 1, j, m), 1, 0, 0) if m <= cap else None
            for i in range(1, j):
                for mp in range(1, min(m - 1, cap) + 1):
                    head = best[i][m - mp]
                    if head is None:
                        continue
                    evals += 1
                    cand = (max(head[0], link[i], stage_time(ctx, i + 1, j, mp)), head[1] + 1, i, mp)
                    if _better(cand, cell):
                        cell = cand
            best[j][m] = cell
    if stats is not None:
        stats["subproblem_evals"] = evals
    if force_all_machines:
        if best[n][budget] is None:
            raise ValidationError(f"no plan uses exactly {budget} machines with replication cap {cap}")
        used = budget
    else:
        used, pick = None, None
        for m in range(1, budget + 1):
            cell = best[n][m]
            if cell is None:
                continue
            if pick is None or cell[0] < pick[0] - TIME_TOL or (
                    cell[0] <= pick[0] + TIME_TOL and (cell[1], m) < (pick[1], used)):
                pick, used = cell, m
        if used is None:
            raise ValidationError("no feasible plan found")
    stages, j, m = [], n, used
    while True:
        cell = best[j][m]
        if cell[2] == 0:
            stages.append(Stage(1, j, m))
            break
        stages.append(Stage(cell[2] + 1, j, cell[3]))
        j, m = cell[2], m - cell[3]
    stages.reverse()
    return Plan(stages=tuple(stages), bottleneck_time=best[n][used][0],
                noam=noam_for(used, stages[0].replication), machines_used=used)
