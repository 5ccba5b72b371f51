"""Per-layer parity report: device executor vs CPU oracle (debug aid)."""
import sys

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_1806_03377_b200 as pd  # noqa: E402
from oracle.pipeline_oracle import mlp_train  # noqa: E402


def main(width=1024, layers=8, stages=4, batch=32, dtype="fp32", lr=2e-4, K=20, mode="weight_stashing"):
    per = layers // stages
    bounds = [(s * per + 1, (s + 1) * per) for s in range(stages)]
    plan = pd.Plan(stages=tuple(pd.Stage(a, b, 1) for a, b in bounds), bottleneck_time=1.0, noam=stages,
                   machines_used=stages)
    cfg = pd.SimConfig(plan=plan, mode=mode, num_minibatches=K)
    spec = pd.mlp(width, layers, batch=batch, dtype=dtype, lr=lr, n_blocks=8, seed=0)
    res = pd.run(cfg, model=spec)
    P = pd.init_params(spec)
    X, T = pd.make_data(spec)
    vers = lambda s, mb, d: res.ledger.version_used(s, mb, pd.Direction(d))  # noqa: E731
    losses, final = mlp_train(P, X, T, lr, bounds, vers, K, emulate="bf16" if dtype == "bf16" else None)
    print("loss rel", np.max(np.abs(np.array(res.losses[:K]) - losses) / losses))
    print("per-step loss rel", np.array2string(np.abs(np.array(res.losses[:K]) - losses) / losses, precision=2))
    for l in range(1, layers + 1):
        Wd, bd = res.weights[l]
        Wo, bo = final[l - 1]
        W0, b0 = P[l - 1]
        dW, dWo = Wd - W0, Wo - W0
        db, dbo = bd - b0, bo - b0
        if not np.any(dWo):
            print(l, "W max|dev-init|", np.abs(dW).max(), "b", np.abs(db).max())
            continue
        print(l, "W delta relerr %.3e" % (np.abs(dW - dWo).max() / np.abs(dWo).max()),
              "b delta relerr %.3e" % (np.abs(db - dbo).max() / np.abs(dbo).max()),
              "ratio |dW|/|dWo| %.4f" % (np.linalg.norm(dW) / np.linalg.norm(dWo)),
              "ratio |db|/|dbo| %.4f" % (np.linalg.norm(db) / np.linalg.norm(dbo)))


if __name__ == "__main__":
    kw = {}
    for a in sys.argv[1:]:
        k, v = a.split("=")
        kw[k] = type(main.__defaults__[list(main.__code__.co_varnames).index(k)])(v)
    main(**kw)
