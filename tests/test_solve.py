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


def test_solve_on_measured_b200_profiles():
    """The planner on B200-measured layer profiles (profiles/layer_profiles, written by
    pd.profile_model): with a 100 Gb/s-class link it reproduces PipeDream's VGG-16 choice on 8
    machines, 7-1; at NVLink bandwidth it prefers data parallelism."""
    import os

    import paper_1806_03377_b200 as pd

    root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "layer_profiles")
    vgg = pd.load_profile(os.path.join(root, "vgg16_profile.json"))
    assert vgg.num_layers == 16 and all(l.fwd_time > 0 and l.bwd_time > 0 for l in vgg.layers)
    plan = pd.solve(pd.build_context(vgg, pd.HardwareSpec(8, 12.5e9, 2)))
    assert [(s.first_layer, s.last_layer, s.replication) for s in plan.stages] == [(1, 13, 7), (14, 16, 1)]
    plan = pd.solve(pd.build_context(vgg, pd.HardwareSpec(8, 770e9, 2)))
    assert [s.replication for s in plan.stages] == [8]
    gpt = pd.load_profile(os.path.join(root, "gpt2_medium_profile.json"))
    plan = pd.solve(pd.build_context(gpt, pd.HardwareSpec(8, 770e9, 2)), max_replication=1)
    assert plan.num_stages == 8 and plan.num_layers == 26
