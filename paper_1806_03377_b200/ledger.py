"""Result types of the executor and the staleness checks (pipesim/simulator.py:37-141, 359-498).

``run()`` returns the same ``SimResult(report, ledger, trace)`` shape as the
reference, except that trace times are measured device timestamps (seconds
from the start of the run) instead of simulated ones, and the report's
throughput/utilisation come from those timestamps with the reference's own
steady-window rule (simulator.py:361-385).
"""

from __future__ import annotations

import csv
from dataclasses import dataclass, field
from enum import Enum
from pathlib import Path

from .errors import SimulationError, ValidationError
from .orders import Direction


class Mode(str, Enum):
    NAIVE_PIPELINE = "naive_pipeline"
    WEIGHT_STASHING = "weight_stashing"
    VERTICAL_SYNC = "vertical_sync"


@dataclass
class SimConfig:
    """Run configuration (simulator.py:43-66); same preconditions."""

    plan: object
    mode: Mode
    num_minibatches: int
    max_inflight: int | None = None
    overlap_comm: bool = True

    def __post_init__(self):
        self.mode = Mode(self.mode)
        if self.max_inflight is not None and not 1 <= self.max_inflight <= self.plan.noam:
            raise ValidationError(f"max_inflight must be within 1..NOAM={self.plan.noam}")
        if self.num_minibatches < self.plan.noam + 10:
            raise ValidationError("num_minibatches must be at least NOAM + 10 to reach steady state")

    @property
    def effective_inflight(self) -> int:
        return self.plan.noam if self.max_inflight is None else self.max_inflight


@dataclass
class VersionLedger:
    """Write-once (stage, minibatch, direction) -> version; v = initial + updates of 1..v."""

    n_stages: int
    stage_replications: tuple[int, ...]
    entries: dict = field(default_factory=dict)
    latest: dict = field(default_factory=dict)

    def record(self, stage: int, minibatch: int, direction: Direction, version: int) -> None:
        key = (stage, minibatch, direction)
        if key in self.entries:
            raise ValidationError(f"ledger entry {key} written twice")
        self.entries[key] = version

    def version_used(self, stage: int, minibatch: int, direction: Direction) -> int:
        return self.entries[(stage, minibatch, direction)]

    @property
    def minibatches(self) -> list[int]:
        return sorted({mb for (_, mb, _) in self.entries})

    @property
    def is_straight(self) -> bool:
        return all(r == 1 for r in self.stage_replications)


@dataclass(frozen=True)
class TraceEvent:
    time_start: float
    time_end: float
    worker: int
    minibatch: int
    stage: int
    direction: Direction
    version_used: int


@dataclass
class SimReport:
    makespan: float
    steady_throughput: float
    per_worker_utilization: tuple[float, ...]
    comm_bytes_total: float
    peak_versions_per_stage: dict
    peak_inflight_per_stage: dict

    def to_dict(self) -> dict:
        return {
            "makespan": self.makespan,
            "steady_throughput": self.steady_throughput,
            "per_worker_utilization": list(self.per_worker_utilization),
            "comm_bytes_total": self.comm_bytes_total,
            "peak_versions_per_stage": {str(k): v for k, v in sorted(self.peak_versions_per_stage.items())},
            "peak_inflight_per_stage": {str(k): v for k, v in sorted(self.peak_inflight_per_stage.items())},
        }


@dataclass
class SimResult:
    report: SimReport
    ledger: VersionLedger
    trace: list
    # B200 additions (absent from the reference's SimResult): per-minibatch losses,
    # final fp32 weights per layer, bubble fraction and executor diagnostics.
    losses: list | None = None
    weights: dict | None = None
    extras: dict = field(default_factory=dict)


@dataclass(frozen=True)
class StalenessViolation:
    stage_index: int
    minibatch_id: int
    direction: Direction
    expected: int
    actual: int


def staleness_check(ledger: VersionLedger, mode, n_stages: int) -> list[StalenessViolation]:
    """Closed-form staleness rules for a straight pipeline at NOAM (simulator.py:423-466).

    stash: stage s (0-based) reads max(0, mb - n + s); vertical sync: max(0, mb - n);
    naive: report every forward/backward disagreement.
    """
    mode = Mode(mode)
    if not ledger.is_straight:
        raise ValidationError(
            f"staleness equations apply to straight pipelines only (replications: {ledger.stage_replications})"
        )
    if n_stages != ledger.n_stages:
        raise ValidationError(f"ledger has {ledger.n_stages} stages, expected {n_stages}")
    out = []
    for mb in ledger.minibatches:
        for s in range(n_stages):
            f = ledger.version_used(s, mb, Direction.FORWARD)
            b = ledger.version_used(s, mb, Direction.BACKWARD)
            if mode is Mode.NAIVE_PIPELINE:
                if f != b:
                    out.append(StalenessViolation(s, mb, Direction.BACKWARD, f, b))
                continue
            want = max(0, mb - n_stages + s) if mode is Mode.WEIGHT_STASHING else max(0, mb - n_stages)
            out.extend(StalenessViolation(s, mb, d, want, got)
                       for d, got in ((Direction.FORWARD, f), (Direction.BACKWARD, b)) if got != want)
    return out


def analytic_throughput(plan) -> float:
    return 1.0 / plan.bottleneck_time


def compare_analytic(report: SimReport, plan) -> float:
    predicted = analytic_throughput(plan)
    return abs(report.steady_throughput - predicted) / predicted


def steady_window(cfg: SimConfig, n_stages: int, input_replication: int) -> tuple[int, int]:
    """Minibatch ids (k1, k2) bounding the steady window (simulator.py:361-375)."""
    inflight_total = cfg.effective_inflight * input_replication
    k1 = inflight_total + n_stages
    k2 = cfg.num_minibatches - inflight_total
    k2 -= (k2 - k1) % input_replication
    if k2 <= k1:
        raise SimulationError(
            f"no steady window: need num_minibatches > {2 * inflight_total + n_stages + input_replication}, "
            f"got {cfg.num_minibatches}"
        )
    return k1, k2


def build_report(cfg: SimConfig, trace: list, n_workers: int, comm_bytes: float) -> SimReport:
    """SimReport from (measured) trace events with the reference's window/utilisation rules."""
    plan = cfg.plan
    n = plan.num_stages
    k1, k2 = steady_window(cfg, n, plan.stages[0].replication)
    completion = {ev.minibatch: ev.time_end for ev in trace
                  if ev.stage == 0 and ev.direction is Direction.BACKWARD}
    t1, t2 = completion[k1], completion[k2]
    span = t2 - t1
    if span <= 0:
        raise SimulationError("steady window has zero duration")
    busy = [0.0] * n_workers
    for ev in trace:
        lo, hi = max(ev.time_start, t1), min(ev.time_end, t2)
        if hi > lo:
            busy[ev.worker] += hi - lo
    # in-flight: +1 at a forward's start, -1 at the matching backward's end (simulator.py:270-275, 317-319)
    deltas = {s: [] for s in range(n)}
    for ev in trace:
        if ev.direction is Direction.FORWARD:
            deltas[ev.stage].append((ev.time_start, 1))
        else:
            deltas[ev.stage].append((ev.time_end, -1))
    peak_inflight = {}
    for s, ds in deltas.items():
        cur = best = 0
        for _, d in sorted(ds, key=lambda x: (x[0], x[1])):
            cur += d
            best = max(best, cur)
        peak_inflight[s] = best
    peak_versions = {s: (1 if cfg.mode is Mode.NAIVE_PIPELINE else peak_inflight[s]) for s in range(n)}
    return SimReport(
        makespan=max((ev.time_end for ev in trace), default=0.0),
        steady_throughput=(k2 - k1) / span,
        per_worker_utilization=tuple(b / span for b in busy),
        comm_bytes_total=float(comm_bytes),
        peak_versions_per_stage=peak_versions,
        peak_inflight_per_stage=peak_inflight,
    )


def write_trace_csv(trace: list, path: str | Path, header_comment: str | None = None) -> None:
    with open(path, "w", newline="") as fh:
        if header_comment:
            fh.write(f"# {header_comment}\n")
        w = csv.writer(fh)
        w.writerow(["time_start", "time_end", "worker", "minibatch", "stage", "direction", "version_used"])
        for ev in trace:
            w.writerow([repr(ev.time_start), repr(ev.time_end), ev.worker, ev.minibatch, ev.stage,
                        ev.direction.value, ev.version_used])
