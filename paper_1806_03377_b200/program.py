"""Compile a 1F1B-RR ``Schedule`` into per-GPU device programs.

The reference resolves readiness, weight versions and transfers at simulated
time inside ``_Engine`` (simulator.py:228-329).  On the B200 every one of those
decisions is a pure function of the static worker orders, so it is resolved
here, on the host, before anything is launched:

* **versions** (simulator.py:228-243, commit at :315): a worker commits version
  ``mb`` when its backward of ``mb`` ends (rep = 1), so a forward reads the id of
  the last backward earlier in the same order.  Stash: the backward reuses it;
  vertical sync: every stage uses the version stage 0's forward read; naive: the
  backward reads the latest at its own start.  For straight pipelines this equals
  the simulator's ledger (tests/test_program.py, golden vectors).  Replicated
  stages (rep > 1) use the round rule of DESIGN.md §5: the k-th backwards of all
  replicas form one allreduce round, after which version k*rep is committed.
* **ring slots** (K7): every version's live range in worker-order positions is
  [commit, last read]; greedy interval colouring gives the minimal ring depth.
* **stash / inbox slots**: activation-stash slot = index of mb in the worker's
  own minibatch list mod cap_s; inbox slots likewise, with the write-after-read
  edge (sender must wait for the previous occupant's backward) made explicit.
* **issue order**: a topological order of the dependency graph (producer edges
  plus the write-after-read edges); a schedule that cannot make progress raises
  ``SimulationError`` naming the blocked worker like simulator.py:345-357.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import SimulationError, ValidationError
from .ledger import Mode, VersionLedger
from .orders import Direction, Schedule, replica_for, stage_inflight_caps

F, B = Direction.FORWARD, Direction.BACKWARD
ITEM_WIDTH = 20  # include/pd_b200.h PD_ITEM_WIDTH


def resolve_versions(schedule: Schedule, mode) -> VersionLedger:
    """Weight version of every pass, from the static orders alone."""
    mode = Mode(mode)
    plan = schedule.plan
    reps = tuple(st.replication for st in plan.stages)
    if mode is Mode.VERTICAL_SYNC and any(r > 1 for r in reps):
        raise ValidationError("vertical_sync is defined for straight pipelines only on the device executor")
    ledger = VersionLedger(n_stages=plan.num_stages, stage_replications=reps)
    fwd_read: dict[tuple[int, int], int] = {}
    latest_after: dict[int, int] = {}
    # pass 1: what each worker's forwards / backwards see of its own commits
    seen: dict[tuple[int, int, Direction], int] = {}
    for wid, order in enumerate(schedule.orders):
        s, _r = schedule.workers[wid]
        rep = reps[s]
        latest, rounds = 0, 0
        for it in order:
            if it.direction is F:
                seen[(s, it.minibatch_id, F)] = latest
            else:
                seen[(s, it.minibatch_id, B)] = latest
                rounds += 1
                latest = it.minibatch_id if rep == 1 else rounds * rep
        latest_after[wid] = latest
    # pass 2: apply the mode's selection rule
    for wid, order in enumerate(schedule.orders):
        s, _r = schedule.workers[wid]
        for it in order:
            mb = it.minibatch_id
            if mode is Mode.VERTICAL_SYNC:
                v = seen[(0, mb, F)]
            elif it.direction is F or mode is Mode.NAIVE_PIPELINE:
                v = seen[(s, mb, it.direction)]
            else:  # stash: backward reuses its forward's version
                v = seen[(s, mb, F)]
            ledger.record(s, mb, it.direction, v)
            if it.direction is F:
                fwd_read[(s, mb)] = v
    for s in range(plan.num_stages):
        ledger.latest[s] = max(latest_after[w] for w, (st, _) in enumerate(schedule.workers) if st == s)
    return ledger


def _color_intervals(intervals: list[tuple[int, int, int]]) -> tuple[dict[int, int], int]:
    """Greedy colouring of (start, end, key) intervals sorted by start; returns key->slot, depth."""
    slot_end: list[int] = []
    assign: dict[int, int] = {}
    for start, end, key in sorted(intervals):
        for i, e in enumerate(slot_end):
            if e < start:
                slot_end[i] = end
                assign[key] = i
                break
        else:
            assign[key] = len(slot_end)
            slot_end.append(end)
    return assign, len(slot_end)


@dataclass
class WorkerPlan:
    """Per-worker resolved program state (one worker = one stage replica = one GPU's share)."""

    wid: int
    stage: int
    replica: int
    mine: list[int]
    cap: int
    ring_slot: dict[int, int] = field(default_factory=dict)  # version -> slot
    ring_depth: int = 1
    act_depth: int = 1
    in_depth: int = 0
    grad_depth: int = 0


@dataclass
class Program:
    schedule: Schedule
    ledger: VersionLedger
    workers: list[WorkerPlan]
    items: list[dict]  # global topological order over all workers
    device_of: list[int]  # worker id -> rank

    def items_for_rank(self, rank: int) -> np.ndarray:
        """int32 [n, ITEM_WIDTH] program for one process; dependency indices are rank-local."""
        mine = [it for it in self.items if self.device_of[it["worker"]] == rank]
        local_index = {it["key"]: i for i, it in enumerate(mine)}
        out = np.full((len(mine), ITEM_WIDTH), -1, dtype=np.int32)
        for i, it in enumerate(mine):
            dep = it["dep"]
            war = it["war"]
            dep_local = dep is not None and self.device_of[dep[0]] == rank
            war_local = war is not None and self.device_of[war[0]] == rank
            op = 0 if it["dir"] is F else (1 if it["dir"] is B else 2)
            out[i] = [
                op, it["stage"], it["mb"], it["worker"], it["version"], it["wslot"],
                it["wnew"], it["act"], it["xslot"], it["gslot"], it["out"], it["block"],
                local_index[dep] if dep_local else -1,
                local_index[war] if war_local else -1,
                it["mb"] if (dep is not None and not dep_local) else 0,
                it["war_mb"] if (war is not None and not war_local) else 0,
                it["dst"], it["src"], it["round"], 0,
            ]
        return out


def compile_program(schedule: Schedule, mode, *, n_blocks: int = 1, world_size: int = 1,
                    device_of: list[int] | None = None) -> Program:
    """Resolve versions, slots and a deadlock-free issue order for ``schedule``."""
    plan = schedule.plan
    n = plan.num_stages
    reps = [st.replication for st in plan.stages]
    caps = stage_inflight_caps(plan, schedule.max_inflight)
    ledger = resolve_versions(schedule, mode)
    W = len(schedule.workers)
    if device_of is None:
        device_of = [min(world_size - 1, (w * world_size) // W) for w in range(W)]
    if len(device_of) != W:
        raise ValidationError(f"device_of has {len(device_of)} entries for {W} workers")

    workers: list[WorkerPlan] = []
    for wid, (s, r) in enumerate(schedule.workers):
        mine = [it.minibatch_id for it in schedule.orders[wid] if it.direction is F]
        workers.append(WorkerPlan(wid, s, r, mine, caps[s]))

    # ---- weight ring slots per worker
    for wp, order in zip(workers, schedule.orders):
        rep = reps[wp.stage]
        commit_pos = {0: -1}
        last_read: dict[int, int] = {}
        rounds = 0
        for p, it in enumerate(order):
            v = ledger.version_used(wp.stage, it.minibatch_id, it.direction)
            last_read[v] = max(last_read.get(v, -1), p)
            if it.direction is B:
                rounds += 1
                commit_pos[it.minibatch_id if rep == 1 else rounds * rep] = p
        intervals = []
        for v, c in commit_pos.items():
            if v in last_read and last_read[v] < c:
                raise ValidationError(f"stage {wp.stage}: version {v} read before it is committed")
            intervals.append((c, max(c, last_read.get(v, c)), v))
        wp.ring_slot, wp.ring_depth = _color_intervals(intervals)
        wp.act_depth = max(1, min(wp.cap, len(wp.mine)))

    def wid_of(s: int, mb: int) -> int:
        return schedule.worker_id(s, replica_for(mb, reps[s]))

    index_in = {wp.wid: {mb: j for j, mb in enumerate(wp.mine)} for wp in workers}
    # inbox depths: activation inbox of stage s+1 holds what stage s may have in flight
    for wp in workers:
        s = wp.stage
        if s > 0:
            wp.in_depth = max(1, min(len(wp.mine), -(-caps[s - 1] * reps[s - 1] // reps[s])))
        if s < n - 1:
            wp.grad_depth = max(1, min(len(wp.mine), wp.cap))

    items: dict[tuple[int, int], dict] = {}
    seqs: list[list[tuple[int, int]]] = []  # per worker: item keys in execution order
    for wp, order in zip(workers, schedule.orders):
        s = wp.stage
        rep = reps[s]
        rounds = 0
        seq = []
        for p, it in enumerate(order):
            mb = it.minibatch_id
            j = index_in[wp.wid].get(mb)
            if j is None:
                raise SimulationError(
                    f"deadlock: worker {wp.wid} (stage {s}, replica {wp.replica}) has a backward of minibatch {mb} "
                    f"without its forward"
                )
            v = ledger.version_used(s, mb, it.direction)
            rec = {
                "key": (wp.wid, len(seq)), "worker": wp.wid, "stage": s, "mb": mb, "dir": it.direction,
                "version": v, "wslot": wp.ring_slot[v], "wnew": -1, "act": j % wp.act_depth, "xslot": -1,
                "gslot": -1, "out": -1, "block": (mb - 1) % n_blocks, "dep": None, "war": None, "war_mb": 0,
                "dst": -1, "src": -1, "round": 0, "xdeps": [],
            }
            if s > 0:
                rec["xslot"] = j % wp.in_depth
            else:
                rec["xslot"] = rec["block"]
            if it.direction is B:
                rounds += 1
                commit_slot = wp.ring_slot[mb if rep == 1 else rounds * rep]
                if s < n - 1:
                    rec["gslot"] = j % wp.grad_depth
                    rec["dep"] = ("B", s + 1, mb)
                    rec["src"] = wid_of(s + 1, mb)
                if s > 0:
                    dst = workers[wid_of(s - 1, mb)]
                    rec["dst"] = dst.wid
                    jd = index_in[dst.wid].get(mb)
                    if jd is None:
                        rec["out"], rec["war"] = 0, ("missing", ("F", s - 1, mb))
                    else:
                        rec["out"] = jd % dst.grad_depth
                        if jd >= dst.grad_depth:
                            rec["war"] = ("B", s - 1, dst.mine[jd - dst.grad_depth])
                # the commit slot: written by this backward (rep 1) or by the round's sharded
                # reduction, which the backward issues layer by layer (rep > 1)
                rec["wnew"] = commit_slot
                if rep > 1:
                    # replicated stage (round rule): the backward only produces this
                    # replica's gradient; a REDUCE item sums all replicas' round-k gradients and commits
                    rec["round"] = rounds
                    if rounds >= 3:  # its gradient buffer (parity k % 2) was read by round k-2
                        rec["xdeps"] = [("R", s, workers[schedule.worker_id(s, r)].mine[rounds - 3])
                                        for r in range(rep) if rounds - 3 < len(workers[schedule.worker_id(s, r)].mine)]
            else:
                if s > 0:
                    rec["dep"] = ("F", s - 1, mb)
                    rec["src"] = wid_of(s - 1, mb)
                if s < n - 1:
                    dst = workers[wid_of(s + 1, mb)]
                    rec["dst"] = dst.wid
                    jd = index_in[dst.wid].get(mb)
                    if jd is None:
                        rec["out"], rec["war"] = 0, ("missing", ("F", s + 1, mb))
                    else:
                        rec["out"] = jd % dst.in_depth
                        if jd >= dst.in_depth:
                            rec["war"] = ("B", s + 1, dst.mine[jd - dst.in_depth])
            items[rec["key"]] = rec
            seq.append(rec["key"])
            if it.direction is B and rep > 1:
                red = dict(rec, key=(wp.wid, len(seq)), dir="R", wnew=commit_slot, dep=None, war=None, war_mb=0,
                           dst=-1, out=-1,
                           xdeps=[("B", s, workers[schedule.worker_id(s, r)].mine[rounds - 1])
                                  for r in range(rep) if rounds - 1 < len(workers[schedule.worker_id(s, r)].mine)])
                items[red["key"]] = red
                seq.append(red["key"])
        seqs.append(seq)

    # resolve symbolic dependencies to item keys
    where = {}
    for key, rec in items.items():
        kind = "F" if rec["dir"] is F else ("B" if rec["dir"] is B else "R")
        where[(kind, rec["stage"], rec["mb"])] = key
    for rec in items.values():
        for k in ("dep", "war"):
            sym = rec[k]
            if sym is None or sym[0] == "missing":
                continue
            if sym not in where:
                rec[k] = ("missing", sym)
            else:
                if k == "war":
                    rec["war_mb"] = sym[2]
                rec[k] = where[sym]
        rec["xdeps"] = [where.get(x, ("missing", x)) for x in rec["xdeps"]]

    # ---- global topological issue order (round-robin list scheduling)
    pos = [0] * W
    done: set = set()
    order_out: list[dict] = []
    total = len(items)
    while len(order_out) < total:
        progressed = False
        for w in range(W):
            while pos[w] < len(seqs[w]):
                rec = items[seqs[w][pos[w]]]
                deps = [d for d in (rec["dep"], rec["war"]) if d is not None] + list(rec["xdeps"])
                if any(d[0] == "missing" or d not in done for d in deps):
                    break
                order_out.append(rec)
                done.add(rec["key"])
                pos[w] += 1
                progressed = True
        if not progressed:
            blocked = [w for w in range(W) if pos[w] < len(seqs[w])]
            w = blocked[0]
            rec = items[seqs[w][pos[w]]]
            s, r = schedule.workers[w]
            what = "reduce" if rec["dir"] == "R" else rec["dir"].value
            raise SimulationError(
                f"deadlock: worker {w} (stage {s}, replica {r}) blocked waiting for {what} of "
                f"minibatch {rec['mb']} ({len(blocked)} workers blocked in total)"
            )
    return Program(schedule=schedule, ledger=ledger, workers=workers, items=order_out, device_of=device_of)
