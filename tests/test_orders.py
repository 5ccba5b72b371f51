"""1F1B-RR schedules and caps: bit-exact against the reference's golden vectors (schedule.py)."""
import pytest

import paper_1806_03377_b200 as pd
from paper_1806_03377_b200.errors import ValidationError
from helpers_golden import compact, load_json, plan_from_stages, reference_pipesim

SCHEDULES = load_json("schedules.json")
CAPS = load_json("caps.json")


@pytest.mark.parametrize("name", sorted(SCHEDULES))
def test_schedule_matches_golden(name):
    g = SCHEDULES[name]
    plan = plan_from_stages(g["stages"])
    sch = pd.build_schedule(plan, g["num_minibatches"], g["max_inflight"])
    assert [list(w) for w in sch.workers] == g["workers"]
    assert [compact(o) for o in sch.orders] == g["orders"]
    assert pd.stage_inflight_caps(plan, g["max_inflight"]) == CAPS[name]
    for wid, (s, r) in enumerate(sch.workers):
        assert sch.worker_id(s, r) == wid


def test_appendix_a1_orders():
    # SURVEY.md Appendix A.1 (cfg1) and test_schedule.py:43-60 known answers
    g = SCHEDULES["straight4_k20"]["orders"]
    assert g[0][:10] == ["F1", "F2", "F3", "F4", "B1", "F5", "B2", "F6", "B3", "F7"]
    assert g[3][:6] == ["F1", "B1", "F2", "B2", "F3", "B3"]
    assert SCHEDULES["vgg_7_1_k28"]["orders"][0] == ["F1", "F8", "B1", "F15", "B8", "F22", "B15", "B22"]


def test_replica_for_and_errors():
    assert pd.replica_for(1, 1) == 0
    assert pd.replica_for(5, 2) == 0
    assert pd.replica_for(6, 2) == 1
    with pytest.raises(ValidationError):
        pd.replica_for(1, 0)
    plan = plan_from_stages([[1, 1, 1], [2, 2, 1]])
    with pytest.raises(ValidationError):
        pd.stage_inflight_caps(plan, max_inflight=3)
    with pytest.raises(ValidationError):
        pd.build_schedule(plan, 0)
    with pytest.raises(ValidationError):
        pd.worker_order(plan, 0, 1, 4)


def test_fifo_backwards_and_forward_first():
    plan = plan_from_stages([[1, 1, 1]] * 1 + [[i, i, 1] for i in range(2, 7)])
    sch = pd.build_schedule(plan, 40)
    for order in sch.orders:
        bwd = [it.minibatch_id for it in order if it.direction is pd.Direction.BACKWARD]
        assert bwd == sorted(bwd)
        seen = set()
        for it in order:
            if it.direction is pd.Direction.FORWARD:
                seen.add(it.minibatch_id)
            else:
                assert it.minibatch_id in seen


def test_schedule_csv(tmp_path):
    plan = plan_from_stages([[1, 1, 1], [2, 2, 1]])
    sch = pd.build_schedule(plan, 12)
    p = tmp_path / "s.csv"
    pd.write_schedule_csv(sch, p, header_comment="x")
    lines = p.read_text().splitlines()
    assert lines[0] == "# x" and lines[1] == "worker,seq,minibatch,stage,direction"
    assert len(lines) == 2 + 2 * 12 * 2


def test_schedule_equals_live_reference():
    ps = reference_pipesim()
    if ps is None:
        pytest.skip("reference package not present (GPU box)")
    for name, g in SCHEDULES.items():
        ref_plan = ps.Plan(stages=tuple(ps.Stage(*s) for s in g["stages"]), bottleneck_time=1.0,
                           noam=ps.noam_for(sum(s[2] for s in g["stages"]), g["stages"][0][2]),
                           machines_used=sum(s[2] for s in g["stages"]))
        ref = ps.build_schedule(ref_plan, g["num_minibatches"], g["max_inflight"])
        mine = pd.build_schedule(ref_plan, g["num_minibatches"], g["max_inflight"])  # duck-typed plan
        assert mine.workers == ref.workers
        assert [[(i.minibatch_id, i.stage_index, i.replica_index, i.direction.value) for i in o] for o in mine.orders] == \
               [[(i.minibatch_id, i.stage_index, i.replica_index, i.direction.value) for i in o] for o in ref.orders]
