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
    model = os.environ.get("PD_MODEL", "mlp")
    n_stages = len(reps)
    K = 20
    if model == "conv":  # VGG-style: conv stack (layers 1-3) and classifier (4-5), PD_REPS = "r0-r1"
        bounds = [(1, 3), (4, 5)]
        layers = (pd.LayerDef("conv", 64), pd.LayerDef("conv", 64, pool=True), pd.LayerDef("conv", 128, pool=True),
                  pd.LayerDef("linear", 32), pd.LayerDef("linear", 16))
        spec = pd.ConvNetSpec(image=(8, 8, 3), layers=layers, batch=16, lr=1e-3, n_blocks=4, seed=0)
    elif model == "gpt":  # GPT-2-style: embedding + block | block + head
        bounds = [(1, 2), (3, 4)]
        spec = pd.GPTSpec(vocab=250, d=256, heads=4, layers=2, seq=128, batch=2, lr=2e-3, n_blocks=3, seed=0)
    else:
        bounds = [(2 * s + 1, 2 * s + 2) for s in range(n_stages)]
        spec = pd.mlp(256, 2 * n_stages, batch=128, dtype="bf16", lr=2e-3, n_blocks=4, seed=3)
    K = K - K % max(reps)
    stages = tuple(pd.Stage(a, b, r) for (a, b), r in zip(bounds, reps))
    used = sum(reps)
    plan = pd.Plan(stages=stages, bottleneck_time=1.0, noam=pd.noam_for(used, reps[0]), machines_used=used)
    cfg = pd.SimConfig(plan=plan, mode="weight_stashing", num_minibatches=K)
    ex = pd.Executor(cfg, model=spec)
    runs = []
    for r in range(3):  # repeated runs exercise the epoch-tagged flags and the end-of-run drain
        torch.distributed.barrier()
        ex.step(trace=(r == 2))
        torch.cuda.synchronize()
        runs.append(ex.result())
    if rank == 0:
        X, T = pd.make_data_any(spec)
        v = lambda s, mb, d: runs[0].ledger.version_used(s, mb, pd.Direction(d))  # noqa: E731
        P = pd.init_params_any(spec)
        worst = 0.0
        for res in runs:
            if model == "conv":
                from oracle.convnet_oracle import convnet_train

                want, P = convnet_train(spec.geoms(), P, X, T, spec.lr, bounds, v, K, reps=reps)
            elif model == "gpt":
                from oracle.gpt_oracle import gpt_train

                want, P = gpt_train(spec, P, X, T, spec.lr, bounds, v, K)
            else:
                from oracle.pipeline_oracle import mlp_train

                want, P = mlp_train(P, X, T, spec.lr, bounds, v, K, emulate="bf16", reps=reps)
            got = np.array(res.losses[:K])
            worst = max(worst, float(np.max(np.abs(got - want) / np.abs(want))))
        rep = runs[-1].report
        # the traced run's ledger is rebuilt from the version tags every rank's passes read on the
        # device; it must equal the program's static resolution exactly
        ledger_ok = runs[-1].extras["ledger_source"] == "device" and \
            runs[-1].ledger.entries == ex.program.ledger.entries
        # payload bytes stored into another process's inbox, counted by the storing kernels, equal
        # the payloads of the program's cross-process hand-offs
        out_feat = [spec.batch * spec.widths[st.last_layer] * spec.bytes_per_elem for st in plan.stages]
        want_bytes = 0
        for it in ex.program.items:
            if it["dir"] == "R" or it["dst"] < 0:
                continue
            if ex.program.device_of[it["dst"]] == ex.program.device_of[it["worker"]]:
                continue
            if it["dir"] is pd.Direction.FORWARD:
                want_bytes += out_feat[it["stage"]]
            else:
                want_bytes += out_feat[it["stage"] - 1]
                if ex.fused_bias(it["stage"] - 1):  # + the receiver's fp32 bias partials [ceil(B/32), width]
                    want_bytes += -(-spec.batch // 32) * spec.widths[plan.stages[it["stage"] - 1].last_layer] * 4
        bytes_ok = runs[-1].extras["p2p_bytes_measured"] == want_bytes
        print(json.dumps({"ok": bool(worst <= 3e-2 and ledger_ok and bytes_ok), "max_rel_loss_err": worst,
                          "ledger_ok": ledger_ok, "p2p_bytes_measured": runs[-1].extras["p2p_bytes_measured"],
                          "p2p_bytes_expected": want_bytes, "world": ex.world, "reps": reps,
                          "model": model,
                          "device_of_worker": runs[-1].extras["device_of_worker"],
                          "bubble": runs[-1].extras["bubble_fraction"],
                          "steady_minibatches_per_s": rep.steady_throughput if rep else None}), flush=True)
    ex.close()
    torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
