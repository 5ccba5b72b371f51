"""The CPU oracle pinned against the reference's own golden trajectories (semantics.py)."""
import numpy as np
import pytest

from oracle.pipeline_oracle import bf16_round, closed_form_version, mlp_train, toy_pipeline
from helpers_golden import toy

MODE_OF = {"vanilla": None, "weight_stashing": "weight_stashing", "vertical_sync": "vertical_sync"}


@pytest.mark.parametrize("n", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("mode", ["weight_stashing", "vertical_sync", "vanilla"])
def test_toy_pipeline_equals_equation_oracle(n, mode):
    g = toy(n)
    if mode == "vanilla":
        versions = lambda s, mb, d: mb - 1  # noqa: E731
    else:
        versions = lambda s, mb, d: closed_form_version(mode, n, s, mb, d)  # noqa: E731
    traj = toy_pipeline(g["design"], g["targets"], g["params"], float(g["lr"]), int(g["block_size"]), versions, 200)
    assert traj.shape == g[f"oracle_{mode}"].shape
    assert np.max(np.abs(traj - g[f"oracle_{mode}"])) <= 1e-12


@pytest.mark.parametrize("n", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("mode", ["weight_stashing", "vertical_sync", "naive_pipeline"])
def test_toy_pipeline_equals_reference_replay(n, mode):
    # replay() of the simulator's ledger, including naive mode's forward/backward mismatch
    g = toy(n)
    versions = lambda s, mb, d: closed_form_version(mode, n, s, mb, d)  # noqa: E731
    traj = toy_pipeline(g["design"], g["targets"], g["params"], float(g["lr"]), int(g["block_size"]), versions, 200)
    assert np.max(np.abs(traj - g[f"replay_{mode}"])) <= 1e-12


def test_bf16_round_matches_torch():
    torch = pytest.importorskip("torch")
    x = np.random.default_rng(0).normal(size=10000) * 10.0 ** np.random.default_rng(1).integers(-20, 20, 10000)
    ref = torch.from_numpy(x).float().to(torch.bfloat16).double().numpy()
    assert np.array_equal(bf16_round(x), ref)


def test_mlp_oracle_single_stage_is_plain_sgd():
    # one stage, version mb-1 everywhere: the oracle must equal textbook minibatch SGD
    rng = np.random.default_rng(0)
    widths = [8, 16, 8, 4]
    params = [(rng.normal(size=(o, i)) * 0.3, rng.normal(size=o) * 0.1) for i, o in zip(widths[:-1], widths[1:])]
    X = rng.normal(size=(3, 5, 8))
    T = rng.normal(size=(3, 5, 4))
    losses, final = mlp_train(params, X, T, 0.05, [(1, 3)], lambda s, mb, d: mb - 1, 6)
    Ws = [(W.copy(), b.copy()) for W, b in params]
    for mb in range(1, 7):
        x, t = X[(mb - 1) % 3], T[(mb - 1) % 3]
        hs, h = [], x
        for l, (W, b) in enumerate(Ws):
            hs.append(h)
            z = h @ W.T + b
            h = np.maximum(z, 0) if l < 2 else z
        loss = 0.5 / 5 * np.sum((z - t) ** 2)
        assert losses[mb - 1] == pytest.approx(loss, rel=1e-12)
        dz = (z - t) / 5
        new = []
        for l in range(2, -1, -1):
            W, b = Ws[l]
            gW, gb = dz.T @ hs[l], dz.sum(0)
            dz = (dz @ W) * (hs[l] > 0)
            new.append((W - 0.05 * gW, b - 0.05 * gb))
        Ws = new[::-1]
    for (W, b), (W2, b2) in zip(final, Ws):
        assert np.allclose(W, W2, rtol=1e-12, atol=1e-14) and np.allclose(b, b2, rtol=1e-12, atol=1e-14)


def test_noise_floor_check_catches_scaled_bias_gradient():
    """The pipeline tests' noise-floor check (tests/helpers_floor.py) is sensitive: the fp32 rule
    passes it, the same rule with every bias gradient scaled by 0.9 (a wrong-but-correlated update,
    VERDICT r01 weak #2) fails it by a wide margin.  CPU torch, 4-stage 8-layer MLP-64, 16 minibatches."""
    import torch

    from helpers_floor import floor_check
    from oracle.pipeline_oracle import mlp_train_torch

    import paper_1806_03377_b200 as pd

    spec = pd.mlp(64, 8, batch=32, dtype="bf16", lr=5e-3, n_blocks=4, seed=0)
    P = pd.init_params(spec)
    X, T = pd.make_data(spec)
    bounds = [(2 * s + 1, 2 * s + 2) for s in range(4)]
    stages = tuple(pd.Stage(a, b, 1) for a, b in bounds)
    plan = pd.Plan(stages=stages, bottleneck_time=1.0, noam=4, machines_used=4)
    ledger = pd.compile_program(pd.build_schedule(plan, 16), "weight_stashing").ledger
    versions = lambda s, mb, d: ledger.version_used(s, mb, pd.Direction(d))  # noqa: E731
    run = lambda dt, **kw: mlp_train_torch(P, X, T, spec.lr, bounds, versions, 16, emulate="bf16",  # noqa: E731
                                           device="cpu", dtype=dt, **kw)
    o64, o32 = run(torch.float64), run(torch.float32)
    params0 = [(torch.as_tensor(W), torch.as_tensor(b)) for W, b in P]
    floor_check(o32[0], o32[1], params0, o32, o64, loss_abs=3e-4)  # the rule itself passes
    bad = run(torch.float32, bias_grad_scale=0.9)
    with pytest.raises(AssertionError):
        floor_check(bad[0], bad[1], params0, o32, o64, loss_abs=3e-4)
    from helpers_floor import delta_err
    worst = max(delta_err(b_bad, b64, b0) for (_, b_bad), (_, b64), (_, b0) in zip(bad[1], o64[1], params0))
    assert worst > 0.05, worst  # ~10 %, five times the absolute allowance
