"""Diagnostic: cfg2 (8 x 2-layer MLP-8192, B=2048, 25 minibatches) device vs the fp64 oracle, next to
the drift of fp32 oracle variants with different summation orders (ksplit 1, 2, 4, 8).
Prints the per-layer training-delta errors.  Usage: python tools/cfg2_floor.py [lr]"""
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
import paper_1806_03377_b200 as pd  # noqa: E402
from oracle.pipeline_oracle import mlp_train_torch  # noqa: E402
from test_fullshape_gpu import _delta_err, _masters, _snapshot, _versions  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False


def main():
    lr = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-5
    K = 25
    stages = tuple(pd.Stage(2 * s + 1, 2 * s + 2, 1) for s in range(8))
    plan = pd.Plan(stages=stages, bottleneck_time=1.0, noam=8, machines_used=8)
    cfg = pd.SimConfig(plan=plan, mode="weight_stashing", num_minibatches=K)
    spec = pd.mlp(8192, 16, batch=2048, dtype="bf16", lr=lr, n_blocks=4, seed=0)
    ex = pd.Executor(cfg, model=spec)
    params0, X, T = _snapshot(ex)
    ex.step(trace=True)
    res = ex.result()
    got = np.array(res.losses[:K])
    dev = [m[0] for _, m in sorted(_masters(ex).items())]
    bounds = [(a.first_layer, a.last_layer) for a in stages]
    w64, f64 = mlp_train_torch(params0, X, T, lr, bounds, _versions(res), K, emulate="bf16", device="cuda",
                               dtype=torch.float64)
    print(f"lr {lr}  env fused_bias={os.environ.get('PD_FUSED_BIAS', '1')} "
          f"conn={os.environ.get('CUDA_DEVICE_MAX_CONNECTIONS')}")
    print("device  loss rel", float(np.max(np.abs(got - w64) / np.abs(w64))))
    print("device  W", [round(_delta_err(W, f[0].float(), p[0]), 4) for (W, _), f, p in zip(dev, f64, params0)])
    print("device  b", [round(_delta_err(b, f[1].float(), p[1]), 4) for (_, b), f, p in zip(dev, f64, params0)])
    for ks in (1, 2, 4, 8):
        w32, f32 = mlp_train_torch(params0, X, T, lr, bounds, _versions(res), K, emulate="bf16", device="cuda",
                                   ksplit=ks)
        print(f"o32 k{ks} loss rel", float(np.max(np.abs(w32 - w64) / np.abs(w64))))
        print(f"o32 k{ks} W", [round(_delta_err(f[0].float(), g[0].float(), p[0]), 4)
                              for f, g, p in zip(f32, f64, params0)])
    ex.close()


if __name__ == "__main__":
    main()
