"""Oracle model ops, fp64 numpy — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper trains "BERT-Large" and "GPT-2" with Adam
 and gives no model internals; this file follows the reading in
SURVEY.md §8(c) Q7/Q8 (listed in DESIGN.md "Readings"):

* pre-LN GPT-2 block: h = LN1(x); qkv = h W_qkv^T + b; o = softmax(q k^T/sqrt(d)
  + mask) v per head; x1 = x + o W_o^T + b_o; h2 = LN2(x1);
  u = gelu_tanh(h2 W_1^T + b_1); x2 = x1 + u W_2^T + b_2.
* causal mask for GPT, none for BERT; LayerNorm eps 1e-5, biased variance.
* learned position embeddings; untied LM head without bias after LN_f.
* loss = mean token cross-entropy over ALL tokens of the step (M*mb*S).
* Adam (not AdamW), bias-corrected, no weight decay / clipping.

Every op has an explicit backward written from its textbook derivative.
Pins: tests/test_oracle_model.py (central finite differences; torch library
routines F.layer_norm / F.gelu / F.scaled_dot_product_attention /
F.cross_entropy / torch.optim.Adam in fp64; closed forms).
"""
import math
import numpy as np

from synth.inputs import param_specs

LN_EPS = 1e-5
GELU_C = math.sqrt(2.0 / math.pi)


# ----------------------------------------------------------------------------
# parameter layout (canonical flat order, synth/inputs.py)
# ----------------------------------------------------------------------------
class Layout:
    """Offsets of every tensor and unit in the canonical flat parameter vector.
    Units: 0 = embedding, 1..L = transformer blocks, L+1 = LN_f + LM head."""

    def __init__(self, m):
        self.m = m
        self.n_units = m.n_layer + 2
        self.entries = []          # (unit, name, shape, offset)
        off = 0
        self.unit_lo = [None] * self.n_units
        self.unit_hi = [None] * self.n_units
        for unit, name, shape, _ in param_specs(m):
            n = int(np.prod(shape))
            if self.unit_lo[unit] is None:
                self.unit_lo[unit] = off
            self.entries.append((unit, name, shape, off))
            off += n
            self.unit_hi[unit] = off
        self.total = off

    def range_of_units(self, a, b):
        """Flat [lo, hi) of units a..b inclusive."""
        return self.unit_lo[a], self.unit_hi[b]

    def tensors(self, flat, lo, hi):
        """Dict name -> reshaped view for the tensors stored in flat[lo:hi]
        (flat is the slice itself, so offsets are rebased by lo)."""
        out = {}
        for _, name, shape, off in self.entries:
            if lo <= off < hi:
                n = int(np.prod(shape))
                out[name] = flat[off - lo: off - lo + n].reshape(shape)
        return out


# ----------------------------------------------------------------------------
# ops (forward returns (out, saved); backward returns input grads + param grads)
# ----------------------------------------------------------------------------
def embedding_fwd(tok_emb, pos_emb, tokens):
    """x[b*S+i] = E[tok[b,i]] + Pos[i]."""
    B, S = tokens.shape
    return tok_emb[tokens.reshape(-1)] + np.tile(pos_emb[:S], (B, 1))


def embedding_bwd(dx, tokens, V, S_max):
    """dE[v] = sum of dx rows whose token is v; dPos[i] = sum over b of dx[b*S+i]."""
    B, S = tokens.shape
    H = dx.shape[1]
    dE = np.zeros((V, H))
    np.add.at(dE, tokens.reshape(-1), dx)
    dPos = np.zeros((S_max, H))
    dPos[:S] = dx.reshape(B, S, H).sum(0)
    return dE, dPos


def layernorm_fwd(x, g, b):
    mu = x.mean(-1, keepdims=True)
    var = ((x - mu) ** 2).mean(-1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + LN_EPS)
    xhat = (x - mu) * rstd
    return xhat * g + b, (xhat, rstd)


def layernorm_bwd(dy, g, saved):
    xhat, rstd = saved
    dxhat = dy * g
    dx = rstd * (dxhat - dxhat.mean(-1, keepdims=True)
                 - xhat * (dxhat * xhat).mean(-1, keepdims=True))
    return dx, (dy * xhat).sum(0), dy.sum(0)


def linear_fwd(x, W, b=None):
    y = x @ W.T
    return y if b is None else y + b


def linear_bwd(dy, x, W):
    """y = x W^T + b  ->  dx = dy W, dW = dy^T x, db = sum_rows dy."""
    return dy @ W, dy.T @ x, dy.sum(0)


def gelu_fwd(x):
    return 0.5 * x * (1.0 + np.tanh(GELU_C * (x + 0.044715 * x ** 3)))


def gelu_bwd(dy, x):
    t = np.tanh(GELU_C * (x + 0.044715 * x ** 3))
    d = 0.5 * (1.0 + t) + 0.5 * x * (1.0 - t * t) * GELU_C * (1.0 + 3 * 0.044715 * x * x)
    return dy * d


def _heads(a, B, S, nh):
    d = a.shape[1] // nh
    return a.reshape(B, S, nh, d).transpose(0, 2, 1, 3)      # [B, nh, S, d]


def _unheads(a):
    B, nh, S, d = a.shape
    return a.transpose(0, 2, 1, 3).reshape(B * S, nh * d)


def attention_fwd(qkv, B, S, nh, causal):
    """Scaled dot-product attention per (sequence, head); qkv columns are
    [q | k | v], head h occupying columns h*d:(h+1)*d of each third."""
    H = qkv.shape[1] // 3
    d = H // nh
    q, k, v = (_heads(qkv[:, i * H:(i + 1) * H], B, S, nh) for i in range(3))
    s = q @ k.transpose(0, 1, 3, 2) / math.sqrt(d)
    if causal:
        s = np.where(np.triu(np.ones((S, S), bool), 1), -np.inf, s)
    s = s - s.max(-1, keepdims=True)
    p = np.exp(s)
    p = p / p.sum(-1, keepdims=True)
    return _unheads(p @ v), p


def attention_bwd(do, qkv, p, B, S, nh):
    H = qkv.shape[1] // 3
    d = H // nh
    q, k, v = (_heads(qkv[:, i * H:(i + 1) * H], B, S, nh) for i in range(3))
    do_ = _heads(do, B, S, nh)
    dv = p.transpose(0, 1, 3, 2) @ do_
    dp = do_ @ v.transpose(0, 1, 3, 2)
    ds = p * (dp - (dp * p).sum(-1, keepdims=True)) / math.sqrt(d)
    dq = ds @ k
    dk = ds.transpose(0, 1, 3, 2) @ q
    return np.concatenate([_unheads(dq), _unheads(dk), _unheads(dv)], axis=1)


def ce_fwd(logits, targets, n_tok):
    """Sum over rows of -log softmax(logits)[target], divided by n_tok (the
    step's total token count, so micro-batch losses add up to the mean)."""
    mx = logits.max(-1, keepdims=True)
    lse = mx + np.log(np.exp(logits - mx).sum(-1, keepdims=True))
    rows = lse[:, 0] - logits[np.arange(len(targets)), targets]
    return rows.sum() / n_tok, np.exp(logits - lse)


def ce_bwd(probs, targets, n_tok):
    d = probs.copy()
    d[np.arange(len(targets)), targets] -= 1.0
    return d / n_tok


def adam_update(p, g, m, v, t, lr, b1, b2, eps):
    """One bias-corrected Adam step ("Adam"); returns new (p, m, v)."""
    m = b1 * m + (1.0 - b1) * g
    v = b2 * v + (1.0 - b2) * g * g
    mhat = m / (1.0 - b1 ** t)
    vhat = v / (1.0 - b2 ** t)
    return p - lr * mhat / (np.sqrt(vhat) + eps), m, v


# ----------------------------------------------------------------------------
# units (embedding / block / head) over one micro-batch
# ----------------------------------------------------------------------------
def unit_fwd(lay, u, th, x, tokens, targets, n_tok):
    """Forward of unit u with parameter views th. Returns (out, saved) where
    out is the activation, or the micro-batch loss for the head unit."""
    m = lay.m
    B, S = tokens.shape
    if u == 0:
        return embedding_fwd(th["tok_emb"], th["pos_emb"], tokens), {}
    if u == m.n_layer + 1:
        h, s_ln = layernorm_fwd(x, th["ln_f.g"], th["ln_f.b"])
        logits = linear_fwd(h, th["w_head"])
        loss, probs = ce_fwd(logits, targets.reshape(-1), n_tok)
        return loss, {"x": x, "h": h, "ln": s_ln, "probs": probs}
    p = f"h{u - 1}."
    h1, s1 = layernorm_fwd(x, th[p + "ln1.g"], th[p + "ln1.b"])
    qkv = linear_fwd(h1, th[p + "w_qkv"], th[p + "b_qkv"])
    o, pr = attention_fwd(qkv, B, S, m.n_head, m.causal)
    x1 = x + linear_fwd(o, th[p + "w_o"], th[p + "b_o"])
    h2, s2 = layernorm_fwd(x1, th[p + "ln2.g"], th[p + "ln2.b"])
    pre = linear_fwd(h2, th[p + "w_1"], th[p + "b_1"])
    act = gelu_fwd(pre)
    x2 = x1 + linear_fwd(act, th[p + "w_2"], th[p + "b_2"])
    return x2, {"x": x, "h1": h1, "s1": s1, "qkv": qkv, "o": o, "p": pr, "x1": x1,
                "h2": h2, "s2": s2, "pre": pre, "act": act}


def unit_bwd(lay, u, th, gr, sv, dout, tokens, targets, n_tok):
    """Backward of unit u. dout is d(loss)/d(unit output) (ignored for the
    head unit, whose output is the loss). Adds parameter gradients into the
    views gr (same names as th) and returns d(loss)/d(unit input), or None
    for the embedding unit."""
    m = lay.m
    B, S = tokens.shape
    if u == 0:
        dE, dP = embedding_bwd(dout, tokens, m.vocab, m.seq_len)
        gr["tok_emb"] += dE
        gr["pos_emb"] += dP
        return None
    if u == m.n_layer + 1:
        dlogits = ce_bwd(sv["probs"], targets.reshape(-1), n_tok)
        dh, dW, _ = linear_bwd(dlogits, sv["h"], th["w_head"])
        gr["w_head"] += dW
        dx, dg, db = layernorm_bwd(dh, th["ln_f.g"], sv["ln"])
        gr["ln_f.g"] += dg
        gr["ln_f.b"] += db
        return dx
    p = f"h{u - 1}."
    dx2 = dout
    dact, dW, db = linear_bwd(dx2, sv["act"], th[p + "w_2"])
    gr[p + "w_2"] += dW
    gr[p + "b_2"] += db
    dpre = gelu_bwd(dact, sv["pre"])
    dh2, dW, db = linear_bwd(dpre, sv["h2"], th[p + "w_1"])
    gr[p + "w_1"] += dW
    gr[p + "b_1"] += db
    dxl, dg, db = layernorm_bwd(dh2, th[p + "ln2.g"], sv["s2"])
    gr[p + "ln2.g"] += dg
    gr[p + "ln2.b"] += db
    dx1 = dx2 + dxl
    do, dW, db = linear_bwd(dx1, sv["o"], th[p + "w_o"])
    gr[p + "w_o"] += dW
    gr[p + "b_o"] += db
    dqkv = attention_bwd(do, sv["qkv"], sv["p"], B, S, m.n_head)
    dh1, dW, db = linear_bwd(dqkv, sv["h1"], th[p + "w_qkv"])
    gr[p + "w_qkv"] += dW
    gr[p + "b_qkv"] += db
    dxl, dg, db = layernorm_bwd(dh1, th[p + "ln1.g"], sv["s1"])
    gr[p + "ln1.g"] += dg
    gr[p + "ln1.b"] += db
    return dx1 + dxl


# ----------------------------------------------------------------------------
# O2: brute-force (unpartitioned, un-microbatched) training step
# ----------------------------------------------------------------------------
def forward_backward(lay, flat, tokens, targets, n_tok=None):
    """Loss and flat gradient of the mean token CE over all given sequences,
    computed over the whole batch at once (no stages, no micro-batches)."""
    n_tok = tokens.size if n_tok is None else n_tok
    th = lay.tensors(flat, 0, lay.total)
    grads = np.zeros(lay.total)
    gr = lay.tensors(grads, 0, lay.total)
    x, saved = None, []
    for u in range(lay.n_units):
        x, sv = unit_fwd(lay, u, th, x, tokens, targets, n_tok)
        saved.append(sv)
    loss = x
    d = None
    for u in reversed(range(lay.n_units)):
        d = unit_bwd(lay, u, th, gr, saved[u], d, tokens, targets, n_tok)
    return loss, grads


def train_step(lay, flat, m_st, v_st, t, tokens, targets, lr, b1, b2, eps):
    """O2: one Adam update of all parameters on the gradient of the mean token
    CE over the step's sequences (SURVEY.md §8(c) "Plain definition")."""
    loss, g = forward_backward(lay, flat, tokens, targets)
    p2, m2, v2 = adam_update(flat, g, m_st, v_st, t, lr, b1, b2, eps)
    return loss, g, p2, m2, v2
