"""Diagnostic: full-shape pipeline parity vs the torch-device oracle across learning rates.
Prints, per lr, the per-minibatch relative loss error and the worst weight-delta error."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_1806_03377_b200 as pd  # noqa: E402
from test_fullshape_gpu import _snapshot, _versions, _masters, _delta_err  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cudnn.allow_tf32 = False


def worst_delta(ex, params0, final):
    m = _masters(ex)
    out = []
    for lid, (W_o, b_o) in enumerate(final, start=1):
        W0, b0 = params0[lid - 1]
        W_d, b_d = m[lid][0]
        out.append((lid, _delta_err(W_d, W_o, W0), _delta_err(b_d, b_o, b0)))
    return out


def run(which, lr):
    if which == "mlp":
        from oracle.pipeline_oracle import mlp_train_torch
        K = 25
        stages = tuple(pd.Stage(2 * s + 1, 2 * s + 2, 1) for s in range(8))
        plan = pd.Plan(stages=stages, bottleneck_time=1.0, noam=8, machines_used=8)
        spec = pd.mlp(8192, 16, batch=2048, dtype="bf16", lr=lr, n_blocks=4, seed=0)
    elif which == "vgg":
        from oracle.convnet_oracle import convnet_train
        K = 42
        plan = pd.Plan(stages=(pd.Stage(1, 13, 7), pd.Stage(14, 16, 1)), bottleneck_time=1.0, noam=2, machines_used=8)
        spec = pd.vgg16(batch=32, lr=lr, n_blocks=2, seed=0)
    else:
        from oracle.gpt_oracle import gpt_train
        K = 12
        spec = pd.GPTSpec(vocab=50257, d=1024, heads=16, layers=2, seq=1024, batch=8, lr=lr, n_blocks=2, seed=0)
        plan = pd.Plan(stages=(pd.Stage(1, 2, 1), pd.Stage(3, 4, 1)), bottleneck_time=1.0, noam=2, machines_used=2)
    cfg = pd.SimConfig(plan=plan, mode="weight_stashing", num_minibatches=K)
    ex = pd.Executor(cfg, model=spec)
    params0, X, T = _snapshot(ex)
    ex.step(trace=True)
    res = ex.result()
    got = np.array(res.losses[:K])
    if which == "mlp":
        want, final = mlp_train_torch(params0, X, T, lr, [(s.first_layer, s.last_layer) for s in plan.stages],
                                      _versions(res), K, emulate="bf16", device="cuda")
    elif which == "vgg":
        want, final = convnet_train(spec.geoms(), params0, X.reshape(X.shape[0], spec.batch, *spec.image), T, lr,
                                    [(1, 13), (14, 16)], _versions(res), K, reps=[7, 1], dtype=torch.float32,
                                    device="cuda")
    else:
        want, final = gpt_train(spec, params0, X, T, lr, [(1, 2), (3, 4)], _versions(res), K, dtype=torch.float32,
                                device="cuda")
    # noise floor: the same rule in fp64 (bf16 rounding points kept); how far an fp32 run drifts
    if which == "mlp":
        w64, f64 = mlp_train_torch(params0, X, T, lr, [(s.first_layer, s.last_layer) for s in plan.stages],
                                   _versions(res), K, emulate="bf16", device="cuda", dtype=torch.float64)
    elif which == "vgg":
        w64, f64 = convnet_train(spec.geoms(), params0, X.reshape(X.shape[0], spec.batch, *spec.image), T, lr,
                                 [(1, 13), (14, 16)], _versions(res), K, reps=[7, 1], dtype=torch.float64,
                                 device="cuda")
    else:
        w64, f64 = gpt_train(spec, params0, X, T, lr, [(1, 2), (3, 4)], _versions(res), K, dtype=torch.float64,
                             device="cuda")
    np.set_printoptions(formatter={"float": lambda v: f"{v:.1e}"})
    print(f"   rel o32 vs o64: {np.abs(want - w64) / np.abs(w64)}")
    print(f"   rel dev vs o64: {np.abs(got - w64) / np.abs(w64)}")
    m = _masters(ex)
    print("   delta err dev-o64 / o32-o64 per layer W:",
          [(lid, round(_delta_err(m[lid][0][0], f64[lid - 1][0].float(), params0[lid - 1][0]), 4),
            round(_delta_err(final[lid - 1][0].float(), f64[lid - 1][0].float(), params0[lid - 1][0]), 4))
           for lid in range(1, len(final) + 1)])
    rel = np.abs(got - want) / np.abs(want)
    print(f"== {which} lr={lr:g}: loss dev[:6]={np.round(got[:6], 4).tolist()} oracle[:6]={np.round(want[:6], 4).tolist()}")
    print(f"   rel per mb: {np.array2string(rel, precision=1, max_line_width=200)}")
    wd = worst_delta(ex, params0, final)
    print("   weight-delta err per layer (W, b):", [(l, round(a, 4), round(b, 4)) for l, a, b in wd])
    ex.close()
    del ex
    torch.cuda.empty_cache()


if __name__ == "__main__":
    for arg in sys.argv[1:]:
        which, lr = arg.split(":")
        run(which, float(lr))
