"""Planner DP: identical plans to the reference's pipesim.solve (partitioner.py:210-308)."""
import pytest

import paper_1806_03377_b200 as pd
from helpers_golden import load_json

CASES = load_json("solve_plans.json")


def ctx_of(case):
    layers = tuple(pd.LayerProfile(i + 1, f"l{i + 1}", f, b, int(a), int(p))
                   for i, (f, b, a, p) in enumerate(case["layers"]))
    return pd.build_context(pd.ModelProfile(layers=layers), pd.HardwareSpec(case["machines"], case["bandwidth"]))


@pytest.mark.parametrize("k", range(len(CASES)))
def test_solve_matches_reference(k):
    case = CASES[k]
    ctx = ctx_of(case)
    if "error" in case["plan"]:
        with pytest.raises(pd.ValidationError):
            pd.solve(ctx, **case["kw"])
        return
    plan = pd.solve(ctx, **case["kw"])
    assert [[s.first_layer, s.last_layer, s.replication] for s in plan.stages] == case["plan"]["stages"]
    assert plan.bottleneck_time == pytest.approx(case["plan"]["bottleneck"], rel=1e-12)
    assert plan.noam == case["plan"]["noam"] and plan.machines_used == case["plan"]["used"]
