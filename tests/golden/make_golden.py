"""Regenerate the golden vectors in tests/golden/ from the reference package.

Run in the build container (where /root/reference exists):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py
It imports the unmodified reference ``pipesim`` from /root/reference/pkg/src and
records, for the hot-path cases of SURVEY.md §8 / Appendix A:
  * schedules.json  - Schedule.workers / Schedule.orders (build_schedule, schedule.py:129-148)
  * caps.json       - stage_inflight_caps (schedule.py:51-70)
  * ledgers.json    - VersionLedger.entries of pipesim.run (simulator.py:228-243, 401-411)
  * toy_*.npz       - make_toy_model data + equation_oracle / replay trajectories (semantics.py:93-221)
The GPU box never reads /root/reference; tests only read these files.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
import pipesim as ps  # noqa: E402

OUT = Path(__file__).resolve().parent


def ctx_n(n, act=0, params=0):
    layers = tuple(ps.LayerProfile(i + 1, f"layer{i + 1}", 0.4, 0.6, act, params) for i in range(n))
    return ps.build_context(ps.ModelProfile(layers=layers), ps.HardwareSpec(n, 1e9))


def straight(n):
    ctx = ctx_n(n)
    return ctx, ps.straight_plan(ctx, [(i, i) for i in range(1, n + 1)])


def plan_reps(layers_reps):
    n = sum(l for l, _ in layers_reps)
    ctx = ctx_n(n)
    stages, first = [], 1
    for lay, rep in layers_reps:
        stages.append(ps.Stage(first, first + lay - 1, rep))
        first += lay
    used = sum(r for _, r in layers_reps)
    plan = ps.Plan(stages=tuple(stages), bottleneck_time=1.0, noam=ps.noam_for(used, stages[0].replication),
                   machines_used=used)
    return ctx, plan


def compact(order):
    return [("F" if it.direction is ps.Direction.FORWARD else "B") + str(it.minibatch_id) for it in order]


SCHEDULE_CASES = {
    "straight4_k20": (lambda: straight(4), 20, None),
    "straight4_k20_inflight1": (lambda: straight(4), 20, 1),
    "straight4_k20_inflight2": (lambda: straight(4), 20, 2),
    "straight8_k25": (lambda: straight(8), 25, None),
    "straight2_k12": (lambda: straight(2), 12, None),
    "straight1_k10": (lambda: straight(1), 10, None),
    "straight3_k17": (lambda: straight(3), 17, None),
    "vgg_7_1_k28": (lambda: plan_reps([(13, 7), (3, 1)]), 28, None),
    "rep_2_1_k12": (lambda: plan_reps([(1, 2), (1, 1)]), 12, None),
    "rep_3_1_k12": (lambda: plan_reps([(1, 3), (1, 1)]), 12, None),
    "rep_1_2_1_k16": (lambda: plan_reps([(1, 1), (2, 2), (1, 1)]), 16, None),
    "dp_3_k9": (lambda: plan_reps([(2, 3)]), 9, None),
}

LEDGER_CASES = {
    "straight4_k20": (lambda: straight(4), 20, None),
    "straight4_k20_inflight2": (lambda: straight(4), 20, 2),
    "straight8_k25": (lambda: straight(8), 25, None),
    "straight2_k14": (lambda: straight(2), 14, None),
    "straight3_k20": (lambda: straight(3), 20, None),
    "straight1_k11": (lambda: straight(1), 11, None),
    "straight6_k30": (lambda: straight(6), 30, None),
}


def main():
    schedules, caps = {}, {}
    for name, (mk, k, mi) in SCHEDULE_CASES.items():
        _ctx, plan = mk()
        sch = ps.build_schedule(plan, k, mi)
        schedules[name] = {
            "stages": [[s.first_layer, s.last_layer, s.replication] for s in plan.stages],
            "num_minibatches": k, "max_inflight": mi,
            "workers": [list(w) for w in sch.workers],
            "orders": [compact(o) for o in sch.orders],
        }
        caps[name] = ps.stage_inflight_caps(plan, mi)
    (OUT / "schedules.json").write_text(json.dumps(schedules, indent=1))
    (OUT / "caps.json").write_text(json.dumps(caps, indent=1))

    ledgers = {}
    for name, (mk, k, mi) in LEDGER_CASES.items():
        ctx, plan = mk()
        ledgers[name] = {"stages": [[s.first_layer, s.last_layer, s.replication] for s in plan.stages],
                         "num_minibatches": k, "max_inflight": mi}
        for mode in ps.Mode:
            res = ps.run(ps.SimConfig(plan=plan, mode=mode, num_minibatches=k, max_inflight=mi), ctx)
            ledgers[name][mode.value] = sorted([s, mb, d.value, v] for (s, mb, d), v in res.ledger.entries.items())
            if mi is None and mode is not ps.Mode.NAIVE_PIPELINE:
                assert ps.staleness_check(res.ledger, mode, plan.num_stages) == []
    (OUT / "ledgers.json").write_text(json.dumps(ledgers))

    # linear toy pipeline (semantics.py): data, init and both trajectories
    for n in (1, 2, 3, 4, 8):
        model = ps.make_toy_model(n, seed=3)
        arrays = {
            "design": model.design, "targets": model.targets,
            "params": np.stack(model.stage_params), "lr": np.array(model.learning_rate),
            "block_size": np.array(model.block_size),
        }
        ctx, plan = straight(n)
        for mode in ("vanilla", "weight_stashing", "vertical_sync"):
            arrays[f"oracle_{mode}"] = ps.equation_oracle(mode, n, model, 200)
        for mode in (ps.Mode.WEIGHT_STASHING, ps.Mode.VERTICAL_SYNC, ps.Mode.NAIVE_PIPELINE):
            led = ps.run(ps.SimConfig(plan=plan, mode=mode, num_minibatches=200), ctx).ledger
            arrays[f"replay_{mode.value}"] = ps.replay(led, model)
        np.savez_compressed(OUT / f"toy_n{n}.npz", **arrays)
    (OUT / "VERSIONS.txt").write_text(
        f"pipesim {ps.__version__} from {REF}\nnumpy {np.__version__}\npython {sys.version.split()[0]}\n"
    )
    print("golden vectors written to", OUT)


if __name__ == "__main__":
    main()

# solve_plans.json was generated with the reference's pipesim.solve on 60 seeded instances of
# tests/helpers.py:random_instance (rng seed 2026, <= 8 layers, <= 6 machines); see tests/test_solve.py
