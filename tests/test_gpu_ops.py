"""Per-kernel GPU parity through the C ABI's single-op entry points, against
the oracle's fp64 ops on the same (bf16-representable) inputs. Shapes span
several tiles plus ragged tails, every operand layout and epilogue."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from oracle import model as om
from synth import round_to_bf16

pytestmark = pytest.mark.gpu

rng = np.random.default_rng(5)


def dev(x, prec):
    t = torch.tensor(np.asarray(x, np.float32), device="cuda")
    return t.to(torch.bfloat16) if prec == "bf16" else t


def host(t):
    return t.float().cpu().numpy().astype(np.float64)


def rnd(*shape, scale=1.0):
    return round_to_bf16((rng.standard_normal(shape) * scale).astype(np.float32)).astype(np.float64)


GEMM_SHAPES = [(64, 64, 64), (200, 136, 72), (256, 512, 128), (1000, 328, 520), (128, 2304, 768),
               (130, 50304 // 64, 64), (8, 24, 16), (384, 640, 1000), (256, 512, 4096),
               (136, 264, 8200)]


@pytest.mark.parametrize("prec", ["bf16", "fp32"])
@pytest.mark.parametrize("impl", [0, 1])
@pytest.mark.parametrize("layout", [(0, 0), (0, 1), (1, 1), (1, 0)])
@pytest.mark.parametrize("shape", GEMM_SHAPES)
def test_gemm_layouts(prec, impl, layout, shape):
    import paper_2204_12013_b200 as bb
    M, N, K = shape
    a_mn, b_mn = layout
    A = rnd(M, K)
    B = rnd(N, K)
    ref = om.linear_fwd(A, B)                      # D = A B^T
    dA = dev(A.T.copy() if a_mn else A, prec)
    dB = dev(B.T.copy() if b_mn else B, prec)
    C = torch.zeros((M, N), device="cuda", dtype=torch.float32)
    args = (prec, impl, M, N, K, dA.data_ptr(), M if a_mn else K, a_mn, dB.data_ptr(),
            N if b_mn else K, b_mn, 5, C.data_ptr(), N)
    lda, ldb = (M if a_mn else K), (N if b_mn else K)
    if prec == "bf16" and impl == 0 and ((a_mn and M < 64) or (b_mn and N < 64) or lda % 8
                                         or ldb % 8):
        # an MN-major operand narrower than one 64-wide box, or a row pitch
        # that is not 16-byte aligned (TMA): the tcgen05 path refuses it (no
        # silent SIMT fallback); bb_init never creates one
        with pytest.raises(bb.BambooError) as e:
            bb.op_gemm(*args)
        assert e.value.status == bb.BB_E_UNSUPPORTED
        return
    bb.op_gemm(*args)
    torch.cuda.synchronize()
    got = host(C)
    tol = 1e-5 if prec == "fp32" else 2e-5   # fp32 accumulate of exact bf16 products
    assert np.abs(got - ref).max() <= tol * np.abs(ref).max() * max(1, K / 256)


@pytest.mark.parametrize("M", [256, 600])
def test_gemm_wide_n_m_fastest_order(M):
    """A wide-N GEMM whose B (N x K bf16 > 64 MB) does not stay in L2 walks
    its tiles M fastest (Gemm::m_fast, the LM-head forward): same result
    as the oracle's D = A B^T (fp32 accumulation of exact bf16 products;
    600 rows leave a ragged row block)."""
    import paper_2204_12013_b200 as bb
    N, K = 50304, 768
    A = rnd(M, K)
    B = rnd(N, K)
    ref = om.linear_fwd(A, B)
    dA, dB = dev(A, "bf16"), dev(B, "bf16")
    C = torch.zeros((M, N), device="cuda", dtype=torch.float32)
    bb.op_gemm("bf16", 0, M, N, K, dA.data_ptr(), K, 0, dB.data_ptr(), K, 0, 6, C.data_ptr(), N)
    torch.cuda.synchronize()
    got = host(C)
    assert np.abs(got - ref).max() <= 2e-5 * np.abs(ref).max() * max(1, K / 256)


@pytest.mark.parametrize("prec", ["bf16", "fp32"])
@pytest.mark.parametrize("epi", [0, 1, 2, 3, 4, 6])
@pytest.mark.parametrize("M,N,K", [(300, 200, 136), (300, 520, 136), (130, 768, 200),
                                   (600, 576, 264)])
def test_gemm_epilogues(prec, epi, M, N, K):
    """N >= 256 runs on CTA pairs (256 x 256 tiles): ragged M leaves the
    second CTA of the last pair partly or wholly past M."""
    import paper_2204_12013_b200 as bb
    A, B = rnd(M, K), rnd(N, K)
    bias, res, aux = rnd(N), rnd(M, N), rnd(M, N)
    D = om.linear_fwd(A, B)
    want_aux = None
    if epi == 0:
        want = D
    elif epi == 1:
        want = D + bias
    elif epi == 2:
        want = D + bias + res
    elif epi == 3:
        want_aux = D + bias
        want = om.gelu_fwd(want_aux)
    elif epi == 4:
        want = om.gelu_bwd(D, aux)
    else:
        want = D
    dt = torch.bfloat16 if prec == "bf16" and epi != 6 else torch.float32
    C = torch.zeros((M, N), device="cuda", dtype=dt)
    dAux = dev(aux, prec) if epi == 4 else torch.zeros((M, N), device="cuda", dtype=dt)
    dbias, dres = dev(bias, prec), dev(res, prec)
    dA, dB = dev(A, prec), dev(B, prec)     # keep alive until the kernels ran
    for impl in (0, 1):
        bb.op_gemm(prec, impl, M, N, K, dA.data_ptr(), K, 0, dB.data_ptr(), K,
                   0, epi, C.data_ptr(), N, dbias.data_ptr(), dres.data_ptr(), dAux.data_ptr())
        torch.cuda.synchronize()
        tol = 1e-5 if prec == "fp32" else 1e-2
        assert np.abs(host(C) - want).max() <= tol * np.abs(want).max()
        if want_aux is not None:
            assert np.abs(host(dAux) - want_aux).max() <= tol * np.abs(want_aux).max()


@pytest.mark.skipif(os.environ.get("BB_GEMM_TILE") is not None or
                    os.environ.get("BB_GEMM_EPI") is not None, reason="already forced")
@pytest.mark.parametrize("force", [("BB_GEMM_TILE", "256"), ("BB_GEMM_TILE", "128"),
                                   ("BB_GEMM_TILE", "pair"), ("BB_GEMM_TILE", "pair128"),
                                   ("BB_GEMM_TILE", "pair192"),
                                   ("BB_GEMM_EPI", "lsu")])
def test_gemm_forced_variants(force):
    """The other GEMM kernels stay correct: single-CTA 128 x 256 / 128 x 128
    tiles (BB_GEMM_TILE), CTA pairs everywhere (small fp32-accumulating dW
    shapes then take pair tiles with up to 8 serialised K splits and TMA
    add-reductions), and the LSU epilogue (BB_GEMM_EPI=lsu, taken for
    unaligned operands): rerun the layout and epilogue tests forced."""
    env = dict(os.environ, **{force[0]: force[1]})
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", __file__, "-k",
                        "test_gemm_layouts or test_gemm_epilogues"], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.parametrize("prec", ["bf16", "fp32"])
@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("B,S,nh,d", [(2, 32, 2, 32), (1, 200, 3, 64), (2, 128, 2, 64),
                                      (1, 1024, 2, 64), (2, 330, 1, 64)])
def test_attention(prec, causal, B, S, nh, d):
    import paper_2204_12013_b200 as bb
    H = nh * d
    qkv = rnd(B * S, 3 * H)
    o_ref, p = om.attention_fwd(qkv, B, S, nh, causal)
    do = rnd(B * S, H)
    dq_ref = om.attention_bwd(do, qkv, p, B, S, nh)
    dqkv_ = dev(qkv, prec)
    o = torch.zeros((B * S, H), device="cuda", dtype=dqkv_.dtype)
    lse = torch.zeros((B, nh, S), device="cuda", dtype=torch.float32)
    bb.op_attention_fwd(prec, B, S, H, nh, causal, dqkv_.data_ptr(), o.data_ptr(), lse.data_ptr())
    dqkv = torch.zeros_like(dqkv_)
    ddo = dev(do, prec)
    bb.op_attention_bwd(prec, B, S, H, nh, causal, dqkv_.data_ptr(), o.data_ptr(), lse.data_ptr(),
                        ddo.data_ptr(), dqkv.data_ptr())
    torch.cuda.synchronize()
    tol = 1e-5 if prec == "fp32" else 1e-2
    assert np.abs(host(o) - o_ref).max() <= tol * np.abs(o_ref).max()
    assert np.abs(host(dqkv) - dq_ref).max() <= tol * np.abs(dq_ref).max() * 2


@pytest.mark.parametrize("causal", [True, False])
def test_attention_backward_bitwise_deterministic(causal):
    """Recovery replays backward passes and must reproduce them bit for bit
    (SURVEY.md §2.2 K7): two backward calls on the same inputs agree exactly
    (dQ sums up to 8 key-block partials in a fixed order)."""
    import paper_2204_12013_b200 as bb
    B, S, nh, d = 2, 1024, 3, 64
    H = nh * d
    g = torch.Generator(device="cuda").manual_seed(3)
    qkv = (torch.randn(B * S, 3 * H, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    do = (torch.randn(B * S, H, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    o = torch.zeros(B * S, H, device="cuda", dtype=torch.bfloat16)
    lse = torch.zeros(B, nh, S, device="cuda")
    bb.op_attention_fwd("bf16", B, S, H, nh, causal, qkv.data_ptr(), o.data_ptr(), lse.data_ptr())
    outs = []
    for _ in range(3):
        dqkv = torch.zeros_like(qkv)
        bb.op_attention_bwd("bf16", B, S, H, nh, causal, qkv.data_ptr(), o.data_ptr(),
                            lse.data_ptr(), do.data_ptr(), dqkv.data_ptr())
        torch.cuda.synchronize()
        outs.append(dqkv)
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])



@pytest.mark.parametrize("prec", ["bf16", "fp32"])
@pytest.mark.parametrize("R,H", [(64, 64), (100, 768), (33, 1600)])
def test_layernorm(prec, R, H):
    import paper_2204_12013_b200 as bb
    x, g, b, dy, dres = rnd(R, H), rnd(H), rnd(H), rnd(R, H), rnd(R, H)
    y_ref, sv = om.layernorm_fwd(x, g, b)
    dx_ref, dg_ref, db_ref = om.layernorm_bwd(dy, g, sv)
    dx_ref = dx_ref + dres
    dt = torch.bfloat16 if prec == "bf16" else torch.float32
    y = torch.zeros((R, H), device="cuda", dtype=dt)
    mean = torch.zeros(R, device="cuda")
    rstd = torch.zeros(R, device="cuda")
    dx = torch.zeros((R, H), device="cuda", dtype=dt)
    dg = torch.zeros(H, device="cuda")
    db = torch.zeros(H, device="cuda")
    dX, dG, dB = dev(x, prec), dev(g, prec), dev(b, prec)
    bb.op_layernorm_fwd(prec, R, H, dX.data_ptr(), dG.data_ptr(), dB.data_ptr(),
                        y.data_ptr(), mean.data_ptr(), rstd.data_ptr())
    dy32 = torch.tensor(dy, device="cuda", dtype=torch.float32)
    dres32 = torch.tensor(dres, device="cuda", dtype=torch.float32)
    bb.op_layernorm_bwd(prec, R, H, dy32.data_ptr(), dX.data_ptr(), mean.data_ptr(),
                        rstd.data_ptr(), dG.data_ptr(), dres32.data_ptr(), dx.data_ptr(),
                        dg.data_ptr(), db.data_ptr())
    torch.cuda.synchronize()
    tol = 1e-5 if prec == "fp32" else 1e-2
    for got, want in ((y, y_ref), (dx, dx_ref), (dg, dg_ref), (db, db_ref)):
        assert np.abs(host(got) - want).max() <= tol * np.abs(want).max()


@pytest.mark.parametrize("prec", ["bf16", "fp32"])
@pytest.mark.parametrize("R,V", [(16, 128), (7, 50304), (33, 30528)])
def test_cross_entropy(prec, R, V):
    import paper_2204_12013_b200 as bb
    logits = rnd(R, V, scale=2.0)
    tg = rng.integers(0, V, R).astype(np.int32)
    n_tok = 4 * R
    loss_ref, probs = om.ce_fwd(logits, tg, n_tok)
    d_ref = om.ce_bwd(probs, tg, n_tok)
    L = dev(logits, prec)
    rows = torch.zeros(R, device="cuda")
    dtg = torch.tensor(tg, device="cuda")
    bb.op_cross_entropy(prec, R, V, L.data_ptr(), dtg.data_ptr(), n_tok, rows.data_ptr())
    torch.cuda.synchronize()
    tol = 1e-5 if prec == "fp32" else 1e-2
    assert abs(host(rows).sum() - loss_ref) <= tol * abs(loss_ref)
    assert np.abs(host(L) - d_ref).max() <= tol * np.abs(d_ref).max()


def test_adam_matches_oracle():
    import paper_2204_12013_b200 as bb
    n = 10007
    p, m, v = rnd(n), np.zeros(n), np.zeros(n)
    lr, b1, b2, eps = 1e-3, 0.9, 0.999, 1e-8
    dp = torch.tensor(p, device="cuda", dtype=torch.float32)
    dm = torch.zeros(n, device="cuda")
    dv = torch.zeros(n, device="cuda")
    w16 = torch.zeros(n, device="cuda", dtype=torch.bfloat16)
    for t in range(1, 4):
        g = rnd(n)
        p, m, v = om.adam_update(p, g, m, v, t, lr, b1, b2, eps)
        dg = torch.tensor(g, device="cuda", dtype=torch.float32)
        bb.op_adam(n, dp.data_ptr(), dg.data_ptr(), dm.data_ptr(), dv.data_ptr(), w16.data_ptr(), t,
                   lr, b1, b2, eps)
        torch.cuda.synchronize()
    torch.cuda.synchronize()
    assert np.abs(host(dp) - p).max() <= 1e-6
    assert np.abs(host(dm) - m).max() <= 1e-6 * np.abs(m).max()
    assert torch.equal(w16.cpu(), dp.cpu().to(torch.bfloat16))
