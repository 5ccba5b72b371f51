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
