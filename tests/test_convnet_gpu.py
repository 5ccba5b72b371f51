"""VGG-style convolutional pipelines (BASELINE configs[2]) on the device against the CPU oracle.

Small network (8x8x3 images; conv64 -> conv64+pool -> conv128+pool -> fc32 -> fc16, softmax
cross-entropy) so the float64 oracle finishes in seconds; the layer kinds, the im2col'ed image
layer, pooling, the stage hand-offs and the replicated-stage round rule are those of VGG-16 7-1.
Tolerances: bf16 storage + fp32 accumulation vs the bf16-emulating fp64 oracle: per-minibatch
loss rel <= 2e-2, per-tensor training-delta Frobenius error <= 1e-1.  Versions are exact.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1806_03377_b200 as pd  # noqa: E402
from oracle.convnet_oracle import convnet_train  # noqa: E402
from paper_1806_03377_b200.models import ConvNetSpec, LayerDef, init_params_any, make_data_any  # noqa: E402

pytestmark = pytest.mark.gpu


def small_spec(batch=16, image=8, lr=1e-3):
    layers = (LayerDef("conv", 64), LayerDef("conv", 64, pool=True), LayerDef("conv", 128, pool=True),
              LayerDef("linear", 32), LayerDef("linear", 16))
    return ConvNetSpec(image=(image, image, 3), layers=layers, batch=batch, lr=lr, n_blocks=4, seed=0)


def make_cfg(stages, K, mode="weight_stashing"):
    plan = pd.Plan(stages=tuple(pd.Stage(a, b, r) for a, b, r in stages), bottleneck_time=1.0,
                   noam=-(-sum(r for _, _, r in stages) // stages[0][2]),
                   machines_used=sum(r for _, _, r in stages))
    return pd.SimConfig(plan=plan, mode=mode, num_minibatches=K)


def delta_err(spec, got, want):
    P0 = init_params_any(spec)
    worst = 0.0
    for l, (W_o, b_o) in enumerate(want, start=1):
        W_d, b_d = got[l]
        for dev, orc, init in ((W_d, W_o, P0[l - 1][0]), (b_d, b_o, P0[l - 1][1])):
            init32 = init.astype(np.float32).astype(np.float64)
            delta = orc - init32
            worst = max(worst, np.linalg.norm((dev - init32) - delta) / max(np.linalg.norm(delta), 1e-30))
    return worst


def check(spec, cfg, res, K):
    X, y = make_data_any(spec)
    bounds = [(st.first_layer, st.last_layer) for st in cfg.plan.stages]
    reps = [st.replication for st in cfg.plan.stages]
    versions = lambda s, mb, d: res.ledger.version_used(s, mb, pd.Direction(d))  # noqa: E731
    want, final = convnet_train(spec.geoms(), init_params_any(spec), X, y, spec.lr, bounds, versions, K,
                                reps=reps)
    got = np.array(res.losses[:K])
    assert np.all(np.isfinite(got))
    rel = np.max(np.abs(got - want) / np.abs(want))
    assert rel <= 2e-2, (rel, got[:6], want[:6])
    err = delta_err(spec, res.weights, final)
    assert err <= 1e-1, err
    return rel, err


@pytest.mark.parametrize("stages", [[(1, 5, 1)], [(1, 3, 1), (4, 5, 1)], [(1, 1, 1), (2, 3, 1), (4, 5, 1)]])
def test_convnet_straight_parity(stages):
    K = 14
    spec = small_spec()
    cfg = make_cfg(stages, K)
    res = pd.run(cfg, None, model=spec)
    n = len(stages)
    if n > 1:
        assert pd.staleness_check(res.ledger, "weight_stashing", n) == []
    check(spec, cfg, res, K)


def test_convnet_replicated_conv_stage():
    """The 7-1 shape at small scale: conv stack replicated 2x (round-rule allreduce), FC stage 1x."""
    K = 12
    spec = small_spec()
    cfg = make_cfg([(1, 3, 2), (4, 5, 1)], K)
    res = pd.run(cfg, None, model=spec)
    check(spec, cfg, res, K)


def test_convnet_trains_and_vsync():
    K = 16
    spec = small_spec(lr=2e-3)
    cfg = make_cfg([(1, 3, 1), (4, 5, 1)], K, mode="vertical_sync")
    res = pd.run(cfg, None, model=spec)
    assert pd.staleness_check(res.ledger, "vertical_sync", 2) == []
    check(spec, cfg, res, K)
