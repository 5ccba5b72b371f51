"""Device-program compilation: versions == reference ledgers, slots, issue order, deadlock."""
import numpy as np
import pytest

import paper_1806_03377_b200 as pd
from paper_1806_03377_b200.errors import SimulationError, ValidationError
from oracle.pipeline_oracle import closed_form_ledger
from helpers_golden import load_json, plan_from_stages

LEDGERS = load_json("ledgers.json")
MODES = ["naive_pipeline", "weight_stashing", "vertical_sync"]


def golden_entries(g, mode):
    return {(s, mb, d): v for s, mb, d, v in g[mode]}


@pytest.mark.parametrize("name", sorted(LEDGERS))
@pytest.mark.parametrize("mode", MODES)
def test_resolved_versions_equal_reference_ledger(name, mode):
    g = LEDGERS[name]
    plan = plan_from_stages(g["stages"])
    sch = pd.build_schedule(plan, g["num_minibatches"], g["max_inflight"])
    led = pd.resolve_versions(sch, mode)
    mine = {(s, mb, d.value): v for (s, mb, d), v in led.entries.items()}
    assert mine == golden_entries(g, mode)


@pytest.mark.parametrize("name", sorted(LEDGERS))
@pytest.mark.parametrize("mode", MODES)
def test_oracle_closed_forms_equal_reference_ledger(name, mode):
    g = LEDGERS[name]
    n = len(g["stages"])
    assert closed_form_ledger(mode, n, g["num_minibatches"], g["max_inflight"]) == golden_entries(g, mode)


@pytest.mark.parametrize("n", [2, 3, 4, 8])
def test_staleness_check_on_resolved_ledgers(n):
    plan = plan_from_stages([[i, i, 1] for i in range(1, n + 1)])
    sch = pd.build_schedule(plan, 3 * n + 10)
    for mode in ("weight_stashing", "vertical_sync"):
        assert pd.staleness_check(pd.resolve_versions(sch, mode), mode, n) == []
    naive = pd.staleness_check(pd.resolve_versions(sch, "naive_pipeline"), "naive_pipeline", n)
    assert {v.minibatch_id for v in naive if v.stage_index == 0} >= set(range(n + 1, 3 * n + 11))


def test_staleness_check_rejects_replicated():
    led = pd.VersionLedger(n_stages=2, stage_replications=(2, 1))
    with pytest.raises(ValidationError):
        pd.staleness_check(led, "weight_stashing", 2)


@pytest.mark.parametrize("n", [1, 2, 4, 8])
@pytest.mark.parametrize("mode", MODES)
def test_ring_depths(n, mode):
    plan = plan_from_stages([[i, i, 1] for i in range(1, n + 1)])
    prog = pd.compile_program(pd.build_schedule(plan, 4 * n + 12), mode)
    caps = pd.stage_inflight_caps(plan)
    for wp in prog.workers:
        if mode == "naive_pipeline":
            assert wp.ring_depth == 2  # latest + the version being written
        elif mode == "weight_stashing":
            assert wp.ring_depth <= caps[wp.stage] + 1  # in-flight stashes + the version being written
        else:
            assert wp.ring_depth <= n + 1  # vertical sync keeps up to n versions + the new one
        assert wp.act_depth == caps[wp.stage]
        # no two simultaneously live versions share a slot
        assert len(set(wp.ring_slot.values())) == wp.ring_depth


def test_issue_order_is_topological_and_complete():
    plan = plan_from_stages([[i, i, 1] for i in range(1, 5)])
    sch = pd.build_schedule(plan, 20)
    prog = pd.compile_program(sch, "weight_stashing")
    arr = prog.items_for_rank(0)
    assert arr.shape == (2 * 4 * 20, pd.program.ITEM_WIDTH)
    for i, row in enumerate(arr):
        assert row[12] < i and row[13] < i  # dep / war issued earlier
        assert row[14] == 0 and row[15] == 0  # single process: no flag waits
    # per-worker subsequences keep the reference order
    for wid, order in enumerate(sch.orders):
        rows = [(int(r[0]), int(r[2])) for r in arr if r[3] == wid]
        assert rows == [(0 if it.direction is pd.Direction.FORWARD else 1, it.minibatch_id) for it in order]


def test_multi_rank_split_uses_flags():
    plan = plan_from_stages([[i, i, 1] for i in range(1, 5)])
    prog = pd.compile_program(pd.build_schedule(plan, 20), "weight_stashing", world_size=2)
    assert prog.device_of == [0, 0, 1, 1]
    r0, r1 = prog.items_for_rank(0), prog.items_for_rank(1)
    assert len(r0) + len(r1) == 160
    # stage 2 forwards (rank 1) wait on the activation flag from stage 1 (rank 0)
    f2 = [r for r in r1 if r[1] == 2 and r[0] == 0]
    assert all(r[12] == -1 and r[14] == r[2] for r in f2)
    # stage 1 backwards (rank 0) wait on stage 2's gradient flag
    b1 = [r for r in r0 if r[1] == 1 and r[0] == 1]
    assert all(r[14] == r[2] for r in b1)
    # stage 1 forwards writing stage 2's inbox wait for the previous occupant's ack once slots recycle
    f1 = [r for r in r0 if r[1] == 1 and r[0] == 0]
    assert [int(r[15]) for r in f1][:4] == [0, 0, 0, 1]


def test_deadlock_names_worker():
    plan = plan_from_stages([[1, 1, 1], [2, 2, 1]])
    sch = pd.build_schedule(plan, 20)
    broken = pd.Schedule(plan=plan, num_minibatches=20, max_inflight=None, workers=sch.workers,
                         orders=((), sch.orders[1]))
    with pytest.raises(SimulationError, match="worker 1"):
        pd.compile_program(broken, "weight_stashing")


def test_config_preconditions():
    plan = plan_from_stages([[i, i, 1] for i in range(1, 5)])
    with pytest.raises(ValidationError):
        pd.SimConfig(plan=plan, mode="weight_stashing", num_minibatches=5)
    with pytest.raises(ValidationError):
        pd.SimConfig(plan=plan, mode="weight_stashing", num_minibatches=20, max_inflight=9)
    cfg = pd.SimConfig(plan=plan, mode="weight_stashing", num_minibatches=20)
    assert cfg.effective_inflight == 4 and cfg.mode is pd.Mode.WEIGHT_STASHING


def test_report_from_synthetic_trace():
    # unit-duration trace of a 2-stage pipeline: window formula as simulator.py:361-385
    plan = plan_from_stages([[1, 1, 1], [2, 2, 1]])
    cfg = pd.SimConfig(plan=plan, mode="weight_stashing", num_minibatches=20)
    trace = [pd.TraceEvent(float(mb), float(mb) + 0.5, 0, mb, 0, pd.Direction.BACKWARD, 0) for mb in range(1, 21)]
    trace += [pd.TraceEvent(float(mb) - 0.5, float(mb), 0, mb, 0, pd.Direction.FORWARD, 0) for mb in range(1, 21)]
    rep = pd.build_report(cfg, trace, 2, 0.0)
    assert rep.steady_throughput == pytest.approx(1.0)
    assert rep.per_worker_utilization[0] == pytest.approx(1.0)
    with pytest.raises(SimulationError, match="steady window"):
        plan8 = plan_from_stages([[i, i, 1] for i in range(1, 9)])
        pd.build_report(pd.SimConfig(plan=plan8, mode="weight_stashing", num_minibatches=18), trace, 8, 0.0)


def test_replicated_program_has_reduce_rounds():
    # 2-1 plan: stage 0 on two replicas (round rule), stage 1 unreplicated
    plan = plan_from_stages([[1, 1, 2], [2, 2, 1]])
    sch = pd.build_schedule(plan, 16)
    prog = pd.compile_program(sch, "weight_stashing")
    arr = prog.items_for_rank(0)
    red = arr[arr[:, 0] == 2]
    bwd0 = arr[(arr[:, 0] == 1) & (arr[:, 1] == 0)]
    assert len(red) == len(bwd0) == 16  # one reduce per replica backward
    # the backward carries its round's commit slot (the sharded reduction it issues writes it); the
    # version is committed (tagged) when the round's reduce item joins the reduction
    assert all(r[18] >= 1 for r in red)
    by_round = {(int(r[3]), int(r[18])): int(r[6]) for r in red}
    assert all(int(b[6]) == by_round[(int(b[3]), int(b[18]))] for b in bwd0)
    # every reduce is issued after both replicas' backwards of its round
    pos = {(int(r[0]), int(r[3]), int(r[18])): i for i, r in enumerate(arr) if r[18] > 0}
    for (op, w, k), i in pos.items():
        if op == 2:
            assert pos[(1, 0, k)] < i and pos[(1, 1, k)] < i
    # forwards after round k read version 2k (replica-summed minibatches 1..2k)
    led = prog.ledger
    assert led.version_used(0, 5, pd.Direction.FORWARD) in (0, 2)
    for wp in prog.workers:
        if wp.stage == 0:
            assert set(wp.ring_slot) >= {0, 2, 4}


def test_replicated_protocol_world2():
    from test_protocol_sim import World

    plan = plan_from_stages([[1, 1, 2], [2, 2, 1]])
    w = World(plan, 16, 2)
    for epoch in (1, 2):
        w.run_epoch(epoch)
