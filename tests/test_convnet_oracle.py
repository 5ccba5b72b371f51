"""The conv-net oracle's hand-written backward equals torch autograd (fp64, no bf16 emulation),
and with one stage and no staleness it is plain SGD on the softmax cross-entropy."""
import numpy as np
import torch

from oracle.convnet_oracle import _backward, _forward, convnet_train
from paper_1806_03377_b200.models import ConvNetSpec, LayerDef, init_params_any, make_data_any


def small_spec(**kw):
    layers = (LayerDef("conv", 64), LayerDef("conv", 64, pool=True), LayerDef("conv", 128, pool=True),
              LayerDef("linear", 32), LayerDef("linear", 16))
    return ConvNetSpec(image=(8, 8, 3), layers=layers, batch=4, **kw)


def test_manual_backward_matches_autograd():
    spec = small_spec()
    geoms = spec.geoms()
    params = init_params_any(spec)
    X, y = make_data_any(spec)
    x = torch.from_numpy(X[0])
    lab = torch.from_numpy(y[0]).long()
    weights = [(torch.from_numpy(W).clone().requires_grad_(True), torch.from_numpy(b).clone().requires_grad_(True))
               for W, b in params]
    with torch.enable_grad():
        logits, _ = _forward(geoms, weights, x, lambda a: a)
        loss = torch.nn.functional.cross_entropy(logits, lab)
        loss.backward()
    with torch.no_grad():
        logits, saved = _forward(geoms, [(W.detach(), b.detach()) for W, b in weights], x, lambda a: a)
        p = torch.softmax(logits, 1)
        p[torch.arange(4), lab] -= 1
        grads = _backward(geoms, [(W.detach(), b.detach()) for W, b in weights], saved, p / 4, lambda a: a)
    for (W, b), (gW, gb) in zip(weights, grads):
        assert torch.allclose(W.grad, gW, rtol=1e-9, atol=1e-12)
        assert torch.allclose(b.grad, gb, rtol=1e-9, atol=1e-12)


def test_single_stage_is_sgd():
    spec = small_spec(lr=0.05)
    geoms = spec.geoms()
    params = init_params_any(spec)
    X, y = make_data_any(spec)
    losses, final = convnet_train(geoms, params, X, y, spec.lr, [(1, 5)], lambda s, mb, d: mb - 1, 3, emulate=None)
    weights = [(torch.from_numpy(W).clone(), torch.from_numpy(b).clone()) for W, b in params]
    for mb in range(1, 4):
        ws = [(W.clone().requires_grad_(True), b.clone().requires_grad_(True)) for W, b in weights]
        with torch.enable_grad():
            logits, _ = _forward(geoms, ws, torch.from_numpy(X[(mb - 1) % 4]), lambda a: a)
            loss = torch.nn.functional.cross_entropy(logits, torch.from_numpy(y[(mb - 1) % 4]).long())
            loss.backward()
        assert abs(loss.item() - losses[mb - 1]) < 1e-12
        weights = [(W.detach() - spec.lr * W.grad, b.detach() - spec.lr * b.grad) for W, b in ws]
    for (W, b), (fW, fb) in zip(weights, final):
        assert np.allclose(W.numpy(), fW, rtol=1e-10, atol=1e-12)
        assert np.allclose(b.numpy(), fb, rtol=1e-10, atol=1e-12)
