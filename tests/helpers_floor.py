"""The noise-floor parity check shared by the pipeline tests.

The reference is the delayed-SGD rule executed in fp64 with bf16 rounding at the device's storage
points; the bound is how far the same rule drifts when executed in fp32 (the floor of any
fp32-accumulating implementation: a bf16 rounding that flips between two fp32 summation orders
compounds through layers and minibatches).  Device distance <= factor x fp32 drift + an absolute
term, per minibatch loss (max relative) and per weight / bias tensor training delta (relative
Frobenius).  The absolute delta term (1e-2) is what makes a wrong-but-correlated update fail:
tests/test_oracle.py::test_noise_floor_check_catches_scaled_bias_gradient shows a bias gradient
scaled by 0.9 exceeding it by a wide margin.
"""
import numpy as np


def delta_err(dev, ref, init):
    """Relative Frobenius error of the training delta (dev - init) against (ref - init)."""
    import torch

    dev, ref, init = ((t if isinstance(t, torch.Tensor) else torch.as_tensor(np.asarray(t))).detach().cpu()
                      for t in (dev, ref, init))
    d_ref = (ref.double() - init.double())
    return float(((dev.double() - init.double()) - d_ref).norm() / max(float(d_ref.norm()), 1e-30))


def floor_check(got_losses, dev_params, params0, o32, o64, loss_abs, delta_abs=1e-2, factor=1.5):
    """Assert the device is within the fp32 noise floor of the fp64 rule.  o32 / o64 = (losses,
    final [(W, b)]) of the oracle in fp32 / fp64; dev_params = [(W, b)] per layer (device).
    Returns (loss rel vs fp64, fp32 drift, rows [(layer, 'W'|'b', device err, fp32 err)])."""
    (w32, f32), (w64, f64) = o32, o64
    got = np.asarray(got_losses, dtype=np.float64)
    rel_dev = float(np.max(np.abs(got - w64) / np.abs(w64)))
    rel_32 = float(np.max(np.abs(np.asarray(w32) - w64) / np.abs(w64)))
    rows = []
    for lid, ((Wd, bd), (W32, b32), (W64, b64), (W0, b0)) in enumerate(zip(dev_params, f32, f64, params0), start=1):
        for name, dev, r32, r64, init in (("W", Wd, W32, W64, W0), ("b", bd, b32, b64, b0)):
            rows.append((lid, name, delta_err(dev, r64, init), delta_err(r32, r64, init)))
    bad = [r for r in rows if not r[2] <= factor * r[3] + delta_abs]
    assert not bad, ("training deltas outside the fp32 noise floor", bad)
    assert np.all(np.isfinite(got)) and rel_dev <= factor * rel_32 + loss_abs, ("loss", rel_dev, rel_32)
    return rel_dev, rel_32, rows
