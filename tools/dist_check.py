"""Multi-process pipeline check: N ranks (one process per GPU, or several on one GPU) run a
4-stage bf16 pipeline with cross-process peer-store inboxes + flags; rank 0 compares the
losses with the CPU oracle and prints one JSON line.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/dist_check.py
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1806_03377_b200 as pd  # noqa: E402


def main():
    backend = os.environ.get("PD_DIST_BACKEND", "gloo")
    torch.distributed.init_process_group(backend)
    rank = torch.distributed.get_rank()
    reps = [int(x) for x in os.environ.get("PD_REPS", "1-1-1-1").split("-")]  # replication per stage
    n_stages = len(reps)
    K = 20
    stages = tuple(pd.Stage(2 * s + 1, 2 * s + 2, r) for s, r in enumerate(reps))
    used = sum(reps)
    plan = pd.Plan(stages=stages, bottleneck_time=1.0, noam=pd.noam_for(used, reps[0]), machines_used=used)
    cfg = pd.SimConfig(plan=plan, mode="weight_stashing", num_minibatches=K)
    spec = pd.mlp(256, 2 * n_stages, batch=128, dtype="bf16", lr=2e-3, n_blocks=4, seed=3)
    ex = pd.Executor(cfg, model=spec)
    runs = []
    for r in range(3):  # repeated runs exercise the epoch-tagged flags and the end-of-run drain
        torch.distributed.barrier()
        ex.step(trace=(r == 2))
        torch.cuda.synchronize()
        runs.append(ex.result())
    if rank == 0:
        from oracle.pipeline_oracle import mlp_train

        X, T = pd.make_data(spec)
        v = lambda s, mb, d: runs[0].ledger.version_used(s, mb, pd.Direction(d))  # noqa: E731
        bounds = [(st.first_layer, st.last_layer) for st in stages]
        P = pd.init_params(spec)
        worst = 0.0
        for res in runs:
            want, P = mlp_train(P, X, T, spec.lr, bounds, v, K, emulate="bf16", reps=reps)
            got = np.array(res.losses[:K])
            worst = max(worst, float(np.max(np.abs(got - want) / np.abs(want))))
        rep = runs[-1].report
        print(json.dumps({"ok": bool(worst <= 3e-2), "max_rel_loss_err": worst, "world": ex.world, "reps": reps,
                          "device_of_worker": runs[-1].extras["device_of_worker"],
                          "bubble": runs[-1].extras["bubble_fraction"],
                          "steady_minibatches_per_s": rep.steady_throughput if rep else None}), flush=True)
    ex.close()
    torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
