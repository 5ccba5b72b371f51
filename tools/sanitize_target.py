"""Small pipelines for compute-sanitizer (memcheck / racecheck / synccheck): one run each of a
4-stage bf16 MLP (tcgen05 GEMMs, fused bias, ring/stash protocol), a 2-1 replicated MLP (round
reduce, graph replay on the second run), a VGG-style 2-1 conv net and a 2-stage GPT-2-style
transformer, each checked against its oracle so a sanitizer-perturbed schedule still has to be right.

    compute-sanitizer --tool memcheck python tools/sanitize_target.py mlp rep conv gpt
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1806_03377_b200 as pd  # noqa: E402


def mlp(reps):
    from oracle.pipeline_oracle import mlp_train

    bounds = [(1, 2), (3, 4)] if reps else [(2 * s + 1, 2 * s + 2) for s in range(4)]
    reps = reps or [1] * 4
    stages = tuple(pd.Stage(a, b, r) for (a, b), r in zip(bounds, reps))
    used = sum(reps)
    plan = pd.Plan(stages=stages, bottleneck_time=1.0, noam=pd.noam_for(used, reps[0]), machines_used=used)
    K = 16
    cfg = pd.SimConfig(plan=plan, mode="weight_stashing", num_minibatches=K)
    spec = pd.mlp(256, 2 * len(bounds), batch=128, dtype="bf16", lr=2e-3, n_blocks=4, seed=0)
    ex = pd.Executor(cfg, model=spec)
    X, T = pd.make_data(spec)
    P = pd.init_params(spec)
    worst = 0.0
    for run in range(2):
        ex.step(trace=(run == 0))
        res = ex.result()
        if run == 0:
            led = res.ledger
        v = lambda s, mb, d: led.version_used(s, mb, pd.Direction(d))  # noqa: E731
        want, P = mlp_train(P, X, T, spec.lr, bounds, v, K, emulate="bf16", reps=reps)
        worst = max(worst, float(np.max(np.abs(np.array(res.losses[:K]) - want) / np.abs(want))))
    ex.close()
    return worst


def main():
    import __graft_entry__ as g

    for what in sys.argv[1:] or ["mlp", "rep", "conv", "gpt"]:
        if what == "mlp":
            r = mlp(None)
        elif what == "rep":
            r = mlp([2, 1])
        elif what == "conv":
            r = g._smoke_convnet()
        else:
            r = g._smoke_gpt()
        print(f"sanitize target {what}: max rel loss err vs oracle {r:.2e}", flush=True)
        assert r <= 3e-2, (what, r)


if __name__ == "__main__":
    main()
