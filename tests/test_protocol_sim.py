"""N>1 hand-off protocol, checked on CPU.

A discrete model of what runtime.cu enqueues for each rank (per-stage streams, event waits for
in-process producers, acquire-polls on inbox/ack flags for peer GPUs, release-signals after each
pass, the end-of-run ack drain) executes the per-rank programs that program.py emits.  It asserts
that no inbox slot is overwritten before its consumer's backward finished, that every read sees
the minibatch it expects, that nothing deadlocks, and that back-to-back runs (epoch-tagged flag
values) stay correct.  The world_size-2 variant exchanges the per-rank programs over a gloo
process group, the same host path the GPU executor uses.
"""
import os

import pytest

import paper_1806_03377_b200 as pd
from helpers_golden import plan_from_stages

FIELDS = dict(op=0, stage=1, mb=2, worker=3, wslot=5, wnew=6, act=7, x=8, g=9, out=10, dep=12, war=13, rwait=14,
              await_=15, dst=16, src=17, round=18)


def f(row, name):
    return int(row[FIELDS[name]])


def enqueue(world, rank, prog, epoch):
    """Per-worker op queues for one rank, mirroring pd_rt_run (receiver-owned flags); a replicated
    worker also has its reduction-stream queue (worker, "R")."""
    queues = {}
    val = lambda mb: epoch * 65536 + mb  # noqa: E731
    last = {}
    for i, row in enumerate(prog):
        w, s, mb, op = f(row, "worker"), f(row, "stage"), f(row, "mb"), f(row, "op")
        fwd = op == 0
        q = queues.setdefault(w, [])
        if f(row, "dep") >= 0:
            q.append(("event", (rank, f(row, "dep"))))
        if f(row, "war") >= 0:
            q.append(("event", (rank, f(row, "war"))))
        if f(row, "rwait") > 0:
            key = ("act_ready", w, f(row, "x")) if fwd else ("grad_ready", w, f(row, "g"))
            q.append(("wait", key, val(f(row, "rwait"))))
        if f(row, "await_") > 0:
            key = ("act_ack" if fwd else "grad_ack", f(row, "dst"), f(row, "out"))
            q.append(("wait", key, val(f(row, "await_"))))
        rep = world.reps[s]
        k = f(row, "round")
        if op == 1 and rep > 1 and k >= 3:
            for r in range(rep):
                q.append(("wait", ("red_done", world.first[s] + r), val(k - 2)))
        if op == 2:  # the reduce item joins the round's reduction stream (runtime.cu run_reduce)
            q.append(("event", ("red", w, k)))
        q.append(("exec", row))
        if op == 1 and rep > 1:
            # sharded reduction, per layer in backward order (runtime.cu issue_layer_reduce): the
            # stage stream signals layer l ready and forks; the reduction stream waits for every
            # replica's layer l, reduce-scatters its shard, signals, waits for every owner, gathers
            rq = queues.setdefault((w, "R"), [])
            for l in range(world.layers[s] - 1, -1, -1):
                q.append(("set", ("lready", w, l), val(k)))
                q.append(("record", ("lev", w, l, k)))
                rq.append(("event", ("lev", w, l, k)))
                rq += [("wait", ("lready", world.first[s] + r, l), val(k)) for r in range(rep)]
                rq.append(("rs", w, s, l, k))
                rq.append(("set", ("lupd", w, l), val(k)))
                rq += [("wait", ("lupd", world.first[s] + r, l), val(k)) for r in range(rep)]
                rq.append(("ag", w, s, l, k))
            rq.append(("set", ("red_done", w), val(k)))
            rq.append(("record", ("red", w, k)))
        q.append(("record", (rank, i)))
        q.append(("signals", row, epoch))
        if op in (0, 1) and f(row, "out") >= 0:
            kk = ("act_ack" if fwd else "grad_ack", f(row, "dst"), f(row, "out"))
            last[(w, kk)] = max(last.get((w, kk), 0), mb)
    return queues, last


class World:
    def __init__(self, plan, K, world, mode="weight_stashing"):
        self.plan = plan
        self.n = plan.num_stages
        self.reps = [st.replication for st in plan.stages]
        self.prog = pd.compile_program(pd.build_schedule(plan, K), mode, world_size=world)
        self.world = world
        self.first = [sum(self.reps[:s]) for s in range(self.n)]
        self.layers = [st.last_layer - st.first_layer + 1 for st in plan.stages]
        self.grads = {}   # (worker, layer, parity) -> round whose gradient the buffer holds
        self.shards = {}  # (stage, layer, owner) -> last round applied by the owner
        self.flags = {}
        self.slots = {}  # (kind, receiver worker, slot) -> [occupant mb, consumed?]
        self.events = set()

    def remote(self, a, b):
        return self.prog.device_of[a] != self.prog.device_of[b]

    def run_epoch(self, epoch):
        queues = {}
        for r in range(self.world):
            q, last = enqueue(self, r, self.prog.items_for_rank(r), epoch)
            for w, ops in q.items():
                # end-of-run drain for outboxes in another process (runtime.cu pd_rt_run)
                for (ww, key), mb in last.items():
                    if ww == w and self.remote(w, key[1]):
                        ops.append(("wait", key, epoch * 65536 + mb))
                queues[(r, w)] = ops
        self.events = set()
        while any(queues.values()):
            progressed = False
            for key, ops in queues.items():
                while ops and self.ready(ops[0]):
                    self.apply(ops.pop(0))
                    progressed = True
            assert progressed, {k: v[0] for k, v in queues.items() if v}

    def ready(self, op):
        if op[0] == "event":
            return op[1] in self.events
        if op[0] == "wait":
            return self.flags.get(op[1], 0) >= op[2]
        return True

    def apply(self, op):
        kind = op[0]
        if kind == "record":
            self.events.add(op[1])
        elif kind == "set":
            self.flags[op[1]] = op[2]
        elif kind == "rs":  # owner w reads every replica's layer-l gradient of round k
            _, w, s, l, k = op
            for r in range(self.reps[s]):
                assert self.grads.get((self.first[s] + r, l, k % 2)) == k, ("reduced a stale gradient", w, l, k)
            self.shards[(s, l, w)] = k
        elif kind == "ag":  # w gathers every owner's round-k shard
            _, w, s, l, k = op
            for r in range(self.reps[s]):
                assert self.shards.get((s, l, self.first[s] + r)) == k, ("gathered a wrong shard", w, l, k)
        elif kind == "exec":
            row = op[1]
            w, s, mb, o = f(row, "worker"), f(row, "stage"), f(row, "mb"), f(row, "op")
            if o == 0:
                if s > 0:
                    occ = self.slots[("act", w, f(row, "x"))]
                    assert occ[0] == mb, ("forward read wrong activation", w, mb, occ)
                if s < self.n - 1:
                    k = ("act", f(row, "dst"), f(row, "out"))
                    assert k not in self.slots or self.slots[k][1], ("activation inbox overwritten", k, mb)
                    self.slots[k] = [mb, False]
            elif o == 1:
                if s > 0:
                    occ = self.slots[("act", w, f(row, "x"))]
                    assert occ[0] == mb
                    occ[1] = True  # stage input no longer needed after the backward (wgrad consumed it)
                if s < self.n - 1:
                    occ = self.slots[("grad", w, f(row, "g"))]
                    assert occ[0] == mb, ("backward read wrong gradient", w, mb, occ)
                    occ[1] = True
                if s > 0:
                    k = ("grad", f(row, "dst"), f(row, "out"))
                    assert k not in self.slots or self.slots[k][1], ("gradient inbox overwritten", k, mb)
                    self.slots[k] = [mb, False]
                if self.reps[s] > 1:  # this replica's round-k gradients land in the parity buffers
                    for l in range(self.layers[s]):
                        self.grads[(w, l, f(row, "round") % 2)] = f(row, "round")
        elif kind == "signals":
            row, epoch = op[1], op[2]
            w, s, mb, o = f(row, "worker"), f(row, "stage"), f(row, "mb"), f(row, "op")
            v = epoch * 65536 + mb
            if o == 0 and s < self.n - 1 and self.remote(w, f(row, "dst")):
                self.flags[("act_ready", f(row, "dst"), f(row, "out"))] = v
            if o == 1 and s > 0 and self.remote(w, f(row, "dst")):
                self.flags[("grad_ready", f(row, "dst"), f(row, "out"))] = v
            if o == 1:  # receiver-owned acks (the runtime signals them when a producer is remote)
                if s > 0:
                    self.flags[("act_ack", w, f(row, "x"))] = v
                if s < self.n - 1:
                    self.flags[("grad_ack", w, f(row, "g"))] = v



@pytest.mark.parametrize("n,world,K", [(4, 2, 20), (8, 2, 25), (8, 4, 25), (8, 8, 25), (3, 2, 16), (4, 4, 14)])
@pytest.mark.parametrize("mode", ["weight_stashing", "vertical_sync", "naive_pipeline"])
def test_protocol_runs_clean_for_three_epochs(n, world, K, mode):
    plan = plan_from_stages([[i, i, 1] for i in range(1, n + 1)])
    w = World(plan, K, world, mode)
    for epoch in (1, 2, 3):
        w.run_epoch(epoch)


def test_protocol_with_max_inflight():
    plan = plan_from_stages([[i, i, 1] for i in range(1, 9)])
    sched = pd.build_schedule(plan, 25, max_inflight=3)
    w = World(plan, 25, 4)
    w.prog = pd.compile_program(sched, "weight_stashing", world_size=4)
    for epoch in (1, 2):
        w.run_epoch(epoch)


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    plan = plan_from_stages([[i, i, 1] for i in range(1, 5)])
    prog = pd.compile_program(pd.build_schedule(plan, 20), "weight_stashing", world_size=world)
    mine = prog.items_for_rank(rank).tolist()
    parts = [None] * world
    dist.all_gather_object(parts, mine)
    dist.destroy_process_group()
    q.put((rank, parts))


def test_world2_gloo_exchange_of_programs():
    """Two gloo ranks exchange their compiled programs; every cross-rank flag wait has a producer."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29400 + os.getpid() % 500
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    parts = got[0]
    assert parts == got[1]
    produced = {(r[1], r[2], r[0]) for part in parts for r in part}
    for rank, part in enumerate(parts):
        for r in part:
            if r[14] > 0:  # waits on a remote producer: forward of stage-1 or backward of stage+1
                src = (r[1] - 1, r[2], 0) if r[0] == 0 else (r[1] + 1, r[2], 1)
                assert src in produced
    assert sum(len(p) for p in parts) == 2 * 4 * 20


@pytest.mark.parametrize("shape,world,K", [([[1, 1, 2], [2, 2, 1]], 1, 16), ([[1, 1, 2], [2, 2, 1]], 3, 16),
                                           ([[1, 1, 1], [2, 2, 2], [3, 3, 1]], 4, 24),
                                           ([[1, 13, 7], [14, 16, 1]], 8, 42)])
def test_protocol_replicated_stages(shape, world, K):
    """Replicated stages: per-round gradient-ready / reduction-done flags, parity buffers (7-1 at 8)."""
    plan = plan_from_stages(shape)
    w = World(plan, K, world)
    for epoch in (1, 2):
        w.run_epoch(epoch)
