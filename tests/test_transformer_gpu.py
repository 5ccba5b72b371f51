"""GPT-2 stage kernels and pipelines (BASELINE configs[3]) on the device.

Kernel tests compare against torch fp32 on the same bf16 inputs (bf16 outputs: |err| <=
2e-2 * max|ref| + 2e-3).  Pipeline tests compare per-minibatch losses with the bf16-emulating
fp64 oracle (oracle/gpt_oracle.py): loss rel <= 1e-2, per-tensor training-delta Frobenius
error <= 1.5e-1 (attention's bf16 P tile and accumulation order are not emulated).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1806_03377_b200 as pd  # noqa: E402
from paper_1806_03377_b200 import _native as nat  # noqa: E402
from paper_1806_03377_b200.models import init_params_any, make_data_any  # noqa: E402

pytestmark = pytest.mark.gpu
F = torch.nn.functional


def _close(got, want, rel=2e-2, floor=2e-3):
    got, want = got.float(), want.float()
    err = (got - want).abs().max().item()
    scale = want.abs().max().item()
    assert err <= rel * scale + floor, f"max err {err:.3e} vs scale {scale:.3e}"


def _ref_attn(qkv, B, S, H):
    d = H * 64
    q, k, v = qkv.float().view(B, S, 3 * d).split(d, dim=-1)
    q, k, v = (t.reshape(B, S, H, 64).transpose(1, 2) for t in (q, k, v))
    return F.scaled_dot_product_attention(q, k, v, is_causal=True)


@pytest.mark.parametrize("B,S,H", [(1, 128, 1), (2, 128, 2), (2, 384, 4), (1, 1024, 16), (8, 1024, 16), (2, 2048, 8)])
def test_attention_fwd_bwd(B, S, H):
    """Forward and the persistent backward vs torch SDPA; (8, 1024, 16) is the GPT-2 bench shape (1 024
    backward items over the SMs, several per CTA), (1, 128, 1) a single item on one CTA."""
    d = 64 * H
    g = torch.Generator(device="cuda").manual_seed(0)
    qkv = torch.randn(B * S, 3 * d, device="cuda", generator=g).bfloat16()
    out = torch.empty(B * S, d, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B, H, S, device="cuda")
    nat.check(nat.lib().pd_attention_fwd(nat.ptr(qkv), nat.ptr(out), nat.ptr(lse), B, S, H, nat.stream_ptr()), "fwd")
    x = qkv.float().clone().requires_grad_(True)
    ref = _ref_attn(x, B, S, H)
    ref_o = ref.transpose(1, 2).reshape(B * S, d)
    torch.cuda.synchronize()
    _close(out, ref_o)
    dout = torch.randn(B * S, d, device="cuda", generator=g).bfloat16()
    ref_o.backward(dout.float())
    dvec = torch.empty(B, H, S, device="cuda")
    dq = torch.empty(B * S, d, device="cuda")
    dqkv = torch.empty(B * S, 3 * d, device="cuda", dtype=torch.bfloat16)
    nat.check(nat.lib().pd_attention_bwd(nat.ptr(qkv), nat.ptr(out), nat.ptr(dout), nat.ptr(lse), nat.ptr(dvec),
                                         nat.ptr(dq), nat.ptr(dqkv), B, S, H, nat.stream_ptr()), "bwd")
    torch.cuda.synchronize()
    for i in range(3):
        _close(dqkv[:, i * d:(i + 1) * d], x.grad[:, i * d:(i + 1) * d], rel=3e-2)


def test_attention_fwd_poly_variant_matches():
    """PD_ATTN_POLY=3 (3 of 8 exp2 pairs on the FMA pipe, degree-3 polynomial) stays within the
    attention tolerance of torch SDPA; run in a child process (the variant is read once per process)."""
    import os
    import subprocess
    import sys
    code = (
        "import sys, torch, paper_1806_03377_b200._native as nat\n"
        "sys.path.insert(0, 'tests')\n"
        "from test_transformer_gpu import _ref_attn, _close\n"
        "B,S,H=2,512,4; d=64*H\n"
        "g=torch.Generator(device='cuda').manual_seed(3)\n"
        "qkv=torch.randn(B*S,3*d,device='cuda',generator=g).bfloat16()\n"
        "out=torch.empty(B*S,d,device='cuda',dtype=torch.bfloat16); lse=torch.empty(B,H,S,device='cuda')\n"
        "nat.check(nat.lib().pd_attention_fwd(nat.ptr(qkv),nat.ptr(out),nat.ptr(lse),B,S,H,nat.stream_ptr()),'fwd')\n"
        "torch.cuda.synchronize()\n"
        "_close(out, _ref_attn(qkv,B,S,H).transpose(1,2).reshape(B*S,d))\n"
        "print('ok')\n")
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=repo, env=dict(os.environ, PD_ATTN_POLY="3"),
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("T,D", [(64, 256), (1000, 1024), (8192, 1024)])
def test_layernorm(T, D):
    g = torch.Generator(device="cuda").manual_seed(1)
    x = (torch.randn(T, D, device="cuda", generator=g) * 2 + 0.5).bfloat16()
    gb = torch.cat([torch.rand(D, device="cuda", generator=g) + 0.5, torch.randn(D, device="cuda", generator=g)])
    y = torch.empty(T, D, device="cuda", dtype=torch.bfloat16)
    mean = torch.empty(T, device="cuda")
    rstd = torch.empty(T, device="cuda")
    nat.check(nat.lib().pd_layernorm_fwd(nat.ptr(x), nat.ptr(gb), nat.ptr(y), nat.ptr(mean), nat.ptr(rstd), T, D,
                                         nat.stream_ptr()), "ln fwd")
    xx = x.float().clone().requires_grad_(True)
    gg = gb[:D].clone().requires_grad_(True)
    bb = gb[D:].clone().requires_grad_(True)
    ref = F.layer_norm(xx, (D,), gg, bb, eps=1e-5)
    torch.cuda.synchronize()
    _close(y, ref)
    dy = torch.randn(T, D, device="cuda", generator=g).bfloat16()
    dres = torch.randn(T, D, device="cuda", generator=g).bfloat16()
    ref.backward(dy.float())
    dx = torch.empty(T, D, device="cuda", dtype=torch.bfloat16)
    nb = nat.lib().pd_layernorm_bwd_blocks(T)
    part = torch.empty(nb, 2 * D, device="cuda")
    nat.check(nat.lib().pd_layernorm_bwd(nat.ptr(dy), nat.ptr(x), nat.ptr(mean), nat.ptr(rstd), nat.ptr(gb),
                                         nat.ptr(dres), nat.ptr(dx), nat.ptr(part), T, D, nat.stream_ptr()), "ln bwd")
    torch.cuda.synchronize()
    _close(dx, xx.grad + dres.float())
    sums = part.sum(0)
    _close(sums[:D], gg.grad, rel=1e-3, floor=1e-2)
    _close(sums[D:], bb.grad, rel=1e-3, floor=1e-2)


def test_embedding_and_vocab_ce():
    V, Vp, S, D, B = 1000, 1024, 64, 256, 3
    T = B * S
    g = torch.Generator(device="cuda").manual_seed(2)
    wte = torch.randn(Vp, D, device="cuda", generator=g).bfloat16()
    wpe = torch.randn(S, D, device="cuda", generator=g).bfloat16()
    tok = torch.randint(0, V, (T,), device="cuda", generator=g, dtype=torch.int32)
    x = torch.empty(T, D, device="cuda", dtype=torch.bfloat16)
    nat.check(nat.lib().pd_embedding_fwd(nat.ptr(tok), nat.ptr(wte), nat.ptr(wpe), nat.ptr(x), T, S, D,
                                         nat.stream_ptr()), "emb")
    pos = torch.arange(T, device="cuda") % S
    ref = wte.float()[tok.long()] + wpe.float()[pos]
    torch.cuda.synchronize()
    _close(x, ref)
    dx = torch.randn(T, D, device="cuda", generator=g).bfloat16()
    gte = torch.zeros(Vp, D, device="cuda")
    gpe = torch.zeros(S, D, device="cuda")
    nat.check(nat.lib().pd_embedding_bwd(nat.ptr(tok), nat.ptr(dx), nat.ptr(gte), nat.ptr(gpe), T, S, D,
                                         nat.stream_ptr()), "emb bwd")
    want_te = torch.zeros(Vp, D, device="cuda").index_add_(0, tok.long(), dx.float())
    want_pe = torch.zeros(S, D, device="cuda").index_add_(0, pos, dx.float())
    torch.cuda.synchronize()
    assert torch.allclose(gte, want_te, atol=1e-4) and torch.allclose(gpe, want_pe, atol=1e-4)
    logits = torch.randn(T, Vp, device="cuda", generator=g) * 2
    logits[:, V:] = 1e4  # padded columns must be ignored
    lab = torch.randint(0, V, (T,), device="cuda", generator=g, dtype=torch.int32)
    dz = torch.empty(T, Vp, device="cuda", dtype=torch.bfloat16)
    loss = torch.zeros(1, device="cuda")
    nat.check(nat.lib().pd_softmax_ce_vocab(nat.ptr(logits), Vp, nat.ptr(lab), T, V, Vp, nat.ptr(dz), Vp,
                                            nat.ptr(loss), nat.stream_ptr()), "ce")
    zz = logits[:, :V].clone().requires_grad_(True)
    ref = F.cross_entropy(zz, lab.long())
    ref.backward()
    torch.cuda.synchronize()
    assert abs(loss.item() - ref.item()) <= 1e-3 * ref.item()
    _close(dz[:, :V], zz.grad)
    assert torch.all(dz[:, V:] == 0)


def test_gelu_resid_epilogues():
    T, K, N = 256, 256, 512
    g = torch.Generator(device="cuda").manual_seed(3)
    A = torch.randn(T, K, device="cuda", generator=g).bfloat16()
    W = (torch.randn(N, K, device="cuda", generator=g) / 16).bfloat16()
    bias = torch.randn(N, device="cuda", generator=g) * 0.1
    u = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
    z = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
    ep = nat.Epilogue(kind=nat.EPI_GELU, out=nat.ptr(u), ldo=N, bias=nat.ptr(bias), aux=nat.ptr(z))
    nat.check(nat.lib().pd_gemm(nat.PD_BF16, nat.ptr(A), 0, K, nat.ptr(W), 0, K, T, N, K, ep, nat.stream_ptr()), "g")
    zr = A.float() @ W.float().T + bias
    torch.cuda.synchronize()
    _close(z, zr)
    _close(u, F.gelu(z.float(), approximate="tanh"))
    # GELU backward: out = acc * gelu'(z)
    dU = torch.randn(T, N, device="cuda", generator=g).bfloat16()
    W2 = (torch.randn(N, N, device="cuda", generator=g) / 16).bfloat16()  # [out=N, in=N]
    out = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
    ep = nat.Epilogue(kind=nat.EPI_GELU_BWD, out=nat.ptr(out), ldo=N, mask=nat.ptr(z), ldm=N)
    nat.check(nat.lib().pd_gemm(nat.PD_BF16, nat.ptr(dU), 0, N, nat.ptr(W2), 1, N, T, N, N, ep, nat.stream_ptr()), "b")
    zz = z.float().clone().requires_grad_(True)
    F.gelu(zz, approximate="tanh").backward(dU.float() @ W2.float())
    torch.cuda.synchronize()
    _close(out, zz.grad)
    # residual: out = acc + bias + resid
    res = torch.randn(T, N, device="cuda", generator=g).bfloat16()
    ep = nat.Epilogue(kind=nat.EPI_RESID, out=nat.ptr(out), ldo=N, bias=nat.ptr(bias), mask=nat.ptr(res), ldm=N)
    nat.check(nat.lib().pd_gemm(nat.PD_BF16, nat.ptr(A), 0, K, nat.ptr(W), 0, K, T, N, K, ep, nat.stream_ptr()), "r")
    torch.cuda.synchronize()
    _close(out, zr + res.float())


def tiny_gpt(**kw):
    base = dict(vocab=250, d=256, heads=4, layers=2, seq=128, batch=2, lr=2e-3, n_blocks=3, seed=0)
    base.update(kw)
    return pd.GPTSpec(**base)


def make_cfg(bounds, K, mode="weight_stashing"):
    stages = tuple(pd.Stage(a, b, 1) for a, b in bounds)
    plan = pd.Plan(stages=stages, bottleneck_time=1.0, noam=len(bounds), machines_used=len(bounds))
    return pd.SimConfig(plan=plan, mode=mode, num_minibatches=K)


def delta_err(spec, got, want):
    P0 = init_params_any(spec)
    worst = {}
    for l, (W_o, b_o) in enumerate(want, start=1):
        W_d, b_d = got[l]
        for name, dev, orc, init in (("W", W_d, W_o, P0[l - 1][0]), ("b", b_d, b_o, P0[l - 1][1])):
            if init.size == 0:
                continue
            i32 = init.astype(np.float32).astype(np.float64)
            dlt = orc.reshape(i32.shape) - i32
            worst[f"{l}{name}"] = np.linalg.norm(dev.reshape(i32.shape) - i32 - dlt) / max(np.linalg.norm(dlt), 1e-30)
    return worst


@pytest.mark.parametrize("bounds", [[(1, 4)], [(1, 2), (3, 4)], [(1, 1), (2, 2), (3, 3), (4, 4)]])
def test_gpt_pipeline_parity(bounds):
    from oracle.gpt_oracle import gpt_train

    K = 14
    spec = tiny_gpt()
    cfg = make_cfg(bounds, K)
    res = pd.run(cfg, None, model=spec)
    if len(bounds) > 1:
        assert pd.staleness_check(res.ledger, "weight_stashing", len(bounds)) == []
    X, y = make_data_any(spec)
    versions = lambda s, mb, d: res.ledger.version_used(s, mb, pd.Direction(d))  # noqa: E731
    want, final = gpt_train(spec, init_params_any(spec), X, y, spec.lr, bounds, versions, K)
    got = np.array(res.losses[:K])
    assert np.all(np.isfinite(got))
    rel = np.max(np.abs(got - want) / np.abs(want))
    assert rel <= 1e-2, (rel, got[:5], want[:5])
    err = delta_err(spec, res.weights, final)
    assert max(err.values()) <= 1.5e-1, err
