"""Pins for oracle/model.py (SURVEY.md §8(c) "What pins each part").

Each op is checked against (a) central finite differences of its own forward
(h=1e-6, fp64) and (b) an independent LIBRARY routine (torch.nn.functional /
torch.optim in float64), plus closed forms. A plausible slip (dropped term,
wrong sign, transposed operand, wrong mask side) fails at least one check.
"""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import model
from synth import get_config, make_params, make_tokens, depth_reduced

rng = np.random.default_rng(0)


def fd_check(f, x, dy, analytic, h=1e-6, n=12, tol=1e-6):
    """Compare <dy, f(x+h e) - f(x-h e)>/(2h) with analytic[e] for n entries."""
    idx = rng.choice(x.size, size=min(n, x.size), replace=False)
    scale = max(1e-12, np.abs(analytic).max())
    for i in idx:
        xp, xm = x.copy(), x.copy()
        xp.flat[i] += h
        xm.flat[i] -= h
        num = (np.sum(dy * f(xp)) - np.sum(dy * f(xm))) / (2 * h)
        assert abs(num - analytic.flat[i]) <= tol * scale + 1e-9, (i, num, analytic.flat[i])


def test_layernorm_fd_and_torch():
    x = rng.standard_normal((6, 16))
    g = rng.standard_normal(16)
    b = rng.standard_normal(16)
    dy = rng.standard_normal((6, 16))
    y, sv = model.layernorm_fwd(x, g, b)
    ref = F.layer_norm(torch.tensor(x), (16,), torch.tensor(g), torch.tensor(b), eps=1e-5)
    assert np.allclose(y, ref.numpy(), rtol=1e-12, atol=1e-12)
    dx, dg, db = model.layernorm_bwd(dy, g, sv)
    fd_check(lambda z: model.layernorm_fwd(z, g, b)[0], x, dy, dx)
    fd_check(lambda z: model.layernorm_fwd(x, z, b)[0], g, dy, dg)
    fd_check(lambda z: model.layernorm_fwd(x, g, z)[0], b, dy, db)
    # closed form: output rows have mean beta-mean... with g=1,b=0: mean 0, var 1/(1+eps/var)
    y1, _ = model.layernorm_fwd(x, np.ones(16), np.zeros(16))
    assert np.allclose(y1.mean(-1), 0, atol=1e-12)


def test_linear_fd():
    x = rng.standard_normal((5, 7))
    W = rng.standard_normal((3, 7))
    b = rng.standard_normal(3)
    dy = rng.standard_normal((5, 3))
    dx, dW, db = model.linear_bwd(dy, x, W)
    assert np.allclose(model.linear_fwd(x, W, b), F.linear(torch.tensor(x), torch.tensor(W),
                                                           torch.tensor(b)).numpy())
    fd_check(lambda z: model.linear_fwd(z, W, b), x, dy, dx)
    fd_check(lambda z: model.linear_fwd(x, z, b), W, dy, dW)
    fd_check(lambda z: model.linear_fwd(x, W, z), b, dy, db)


def test_gelu_tanh_torch_and_fd():
    x = rng.standard_normal(50) * 3
    ref = F.gelu(torch.tensor(x), approximate="tanh").numpy()
    assert np.allclose(model.gelu_fwd(x), ref, rtol=1e-13, atol=1e-14)
    dy = rng.standard_normal(50)
    fd_check(model.gelu_fwd, x, dy, model.gelu_bwd(dy, x), n=50)
    # closed form: gelu(0) = 0, gelu'(0) = 1/2
    assert model.gelu_fwd(np.array([0.0]))[0] == 0.0
    assert model.gelu_bwd(np.array([1.0]), np.array([0.0]))[0] == 0.5


@pytest.mark.parametrize("causal", [True, False])
def test_attention_torch_and_fd(causal):
    B, S, nh, d = 2, 5, 3, 4
    H = nh * d
    qkv = rng.standard_normal((B * S, 3 * H))
    o, p = model.attention_fwd(qkv, B, S, nh, causal)
    t = torch.tensor(qkv).reshape(B, S, 3, nh, d).permute(2, 0, 3, 1, 4)
    ref = F.scaled_dot_product_attention(t[0], t[1], t[2], is_causal=causal)
    ref = ref.permute(0, 2, 1, 3).reshape(B * S, H).numpy()
    assert np.allclose(o, ref, rtol=1e-12, atol=1e-12)
    do = rng.standard_normal((B * S, H))
    dqkv = model.attention_bwd(do, qkv, p, B, S, nh)
    fd_check(lambda z: model.attention_fwd(z, B, S, nh, causal)[0], qkv, do, dqkv, n=40)
    if causal:   # future tokens never influence earlier positions
        q2 = qkv.copy()
        q2.reshape(B, S, 3 * H)[:, -1, :] += 1.0
        o2, _ = model.attention_fwd(q2, B, S, nh, True)
        assert np.array_equal(o2.reshape(B, S, H)[:, :-1], o.reshape(B, S, H)[:, :-1])


def test_cross_entropy_torch_closed_form():
    logits = rng.standard_normal((7, 11)) * 2
    tg = rng.integers(0, 11, 7)
    loss, probs = model.ce_fwd(logits, tg, 7)
    ref = F.cross_entropy(torch.tensor(logits), torch.tensor(tg))
    assert abs(loss - ref.item()) < 1e-13
    d = model.ce_bwd(probs, tg, 7)
    onehot = np.eye(11)[tg]
    sm = torch.softmax(torch.tensor(logits), -1).numpy()
    assert np.allclose(d, (sm - onehot) / 7, atol=1e-15)
    # uniform logits -> loss = log V
    l0, _ = model.ce_fwd(np.zeros((3, 11)), np.array([0, 5, 10]), 3)
    assert abs(l0 - math.log(11)) < 1e-14


def test_embedding_fd():
    V, S, H = 9, 4, 3
    E = rng.standard_normal((V, H))
    Pos = rng.standard_normal((S, H))
    tok = np.array([[1, 1, 8, 0], [3, 1, 2, 2]])
    dx = rng.standard_normal((8, H))
    dE, dP = model.embedding_bwd(dx, tok, V, S)
    fd_check(lambda z: model.embedding_fwd(z, Pos, tok), E, dx, dE, n=27)
    fd_check(lambda z: model.embedding_fwd(E, z, tok), Pos, dx, dP, n=12)


def test_adam_torch_and_closed_form():
    p = rng.standard_normal(20)
    lr, b1, b2, eps = 1e-3, 0.9, 0.999, 1e-8
    tp = torch.tensor(p.copy(), requires_grad=True)
    opt = torch.optim.Adam([tp], lr=lr, betas=(b1, b2), eps=eps)
    m = np.zeros(20)
    v = np.zeros(20)
    cur = p.copy()
    for t in range(1, 4):
        g = rng.standard_normal(20)
        tp.grad = torch.tensor(g)
        opt.step()
        if t == 1:   # closed form of the first bias-corrected step
            expect = cur - lr * g / (np.abs(g) + eps)
        cur, m, v = model.adam_update(cur, g, m, v, t, lr, b1, b2, eps)
        if t == 1:
            assert np.allclose(cur, expect, rtol=0, atol=1e-15)
        assert np.allclose(cur, tp.detach().numpy(), rtol=0, atol=1e-14)


def _torch_model_loss(cfg, flat, tokens, targets):
    """Reference forward composed ONLY of torch library ops (float64)."""
    m = cfg.model
    lay = model.Layout(m)
    P = torch.tensor(flat, requires_grad=True)
    th = {name: P[off:off + int(np.prod(shape))].reshape(shape)
          for _, name, shape, off in lay.entries}
    B, S = tokens.shape
    H, nh = m.d_model, m.n_head
    d = H // nh
    tok = torch.tensor(tokens, dtype=torch.long)
    x = F.embedding(tok, th["tok_emb"]) + th["pos_emb"][:S]
    for layer in range(m.n_layer):
        p = f"h{layer}."
        h = F.layer_norm(x, (H,), th[p + "ln1.g"], th[p + "ln1.b"], 1e-5)
        qkv = F.linear(h, th[p + "w_qkv"], th[p + "b_qkv"]).reshape(B, S, 3, nh, d)
        q, k, v = qkv.permute(2, 0, 3, 1, 4)
        o = F.scaled_dot_product_attention(q, k, v, is_causal=m.causal)
        o = o.permute(0, 2, 1, 3).reshape(B, S, H)
        x = x + F.linear(o, th[p + "w_o"], th[p + "b_o"])
        h = F.layer_norm(x, (H,), th[p + "ln2.g"], th[p + "ln2.b"], 1e-5)
        x = x + F.linear(F.gelu(F.linear(h, th[p + "w_1"], th[p + "b_1"]), approximate="tanh"),
                         th[p + "w_2"], th[p + "b_2"])
    h = F.layer_norm(x, (H,), th["ln_f.g"], th["ln_f.b"], 1e-5)
    logits = F.linear(h, th["w_head"])
    loss = F.cross_entropy(logits.reshape(B * S, -1), torch.tensor(targets.reshape(-1),
                                                                   dtype=torch.long))
    loss.backward()
    return loss.item(), P.grad.numpy()


@pytest.mark.parametrize("name", ["C0", "C2-like"])
def test_full_model_vs_torch_autograd(name):
    if name == "C0":
        cfg = get_config("C0")
    else:   # bidirectional (BERT) variant at tiny width
        import dataclasses
        c0 = get_config("C0")
        cfg = dataclasses.replace(c0, model=dataclasses.replace(c0.model, causal=False), gpt=False)
    flat = make_params(cfg.model).astype(np.float64)
    flat += rng.standard_normal(flat.size) * 1e-2     # non-trivial biases / LN params
    tokens, targets = make_tokens(cfg)
    lay = model.Layout(cfg.model)
    loss, g = model.forward_backward(lay, flat, tokens, targets)
    ref_loss, ref_g = _torch_model_loss(cfg, flat, tokens, targets)
    assert abs(loss - ref_loss) <= 1e-12 * abs(ref_loss)
    assert np.abs(g - ref_g).max() <= 1e-10 * np.abs(ref_g).max()


def test_zero_weights_loss_is_log_vocab():
    cfg = get_config("C0")
    lay = model.Layout(cfg.model)
    flat = np.zeros(lay.total)
    tokens, targets = make_tokens(cfg)
    loss, _ = model.forward_backward(lay, flat, tokens, targets)
    assert abs(loss - math.log(cfg.model.vocab)) < 1e-12


def test_full_model_fd_spot():
    cfg = depth_reduced("C0", 1, 2, 1)
    lay = model.Layout(cfg.model)
    flat = make_params(cfg.model).astype(np.float64)
    tokens, targets = make_tokens(cfg)
    loss, g = model.forward_backward(lay, flat, tokens, targets)
    h = 1e-6
    for i in rng.choice(lay.total, 25, replace=False):
        fp, fm = flat.copy(), flat.copy()
        fp[i] += h
        fm[i] -= h
        num = (model.forward_backward(lay, fp, tokens, targets)[0]
               - model.forward_backward(lay, fm, tokens, targets)[0]) / (2 * h)
        assert abs(num - g[i]) <= 1e-6 * np.abs(g).max() + 1e-10
