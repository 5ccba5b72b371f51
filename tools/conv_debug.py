"""Per-layer training-delta error of a single-stage conv net vs the oracle (debug aid)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_1806_03377_b200 as pd  # noqa: E402
from oracle.convnet_oracle import convnet_train  # noqa: E402
from paper_1806_03377_b200.models import init_params_any, make_data_any  # noqa: E402
from test_convnet_gpu import make_cfg, small_spec  # noqa: E402

lr = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-4
K = 11
spec = small_spec(lr=lr)
cfg = make_cfg([(1, 5, 1)], K)
res = pd.run(cfg, None, model=spec)
X, y = make_data_any(spec)
P0 = init_params_any(spec)
want, final = convnet_train(spec.geoms(), P0, X, y, lr, [(1, 5)], lambda s, mb, d: mb - 1, K)
print("loss dev", np.round(res.losses[:K], 5))
print("loss orc", np.round(want, 5))
for l, (W_o, b_o) in enumerate(final, start=1):
    W_d, b_d = res.weights[l]
    for name, dev, orc, init in (("W", W_d, W_o, P0[l - 1][0]), ("b", b_d, b_o, P0[l - 1][1])):
        i32 = init.astype(np.float32).astype(np.float64)
        d = orc - i32
        e = np.linalg.norm((dev - i32) - d) / max(np.linalg.norm(d), 1e-30)
        print(l, name, f"delta-err {e:.3e}  |delta| {np.linalg.norm(d):.3e} |dev delta| {np.linalg.norm(dev - i32):.3e}")
