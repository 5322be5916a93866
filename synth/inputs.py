"""Seeded synthetic tokens and initial weights (SURVEY.md §8(d) "Synthetic inputs").

* Tokens: numpy PCG64(1234 + config_index + 1000*step). GPT configs draw
  [M*mb, S+1] uniform in [0, vocab_sample) and use [:, :S] as tokens and
  [:, 1:] as targets; BERT draws tokens and targets independently.
* Weights: seed 42; N(0, 0.02) for embeddings, W_qkv, W_1, W_head;
  N(0, 0.02/sqrt(2L)) for W_o, W_2; biases 0; LayerNorm gamma 1, beta 0.
  Every value is rounded to a bf16-representable fp32
  so that the bf16 working copy on the GPU and the fp64 oracle start from
  the same numbers.

The canonical flat parameter order (the layout both sides agree on, see
include/bamboo.h) is: tok_emb[V,H], pos_emb[S,H], then per layer
ln1.g[H], ln1.b[H], w_qkv[3H,H], b_qkv[3H], w_o[H,H], b_o[H], ln2.g[H],
ln2.b[H], w_1[F,H], b_1[F], w_2[H,F], b_2[H], then ln_f.g[H], ln_f.b[H],
w_head[V,H].
"""
import math
import numpy as np

from .configs import ModelCfg, RunCfg


def param_specs(m: ModelCfg):
    """[(unit, name, shape, init)] in canonical order; unit 0 = embedding,
    1..L = blocks, L+1 = head. init in {'emb','w','wres','zero','one'}."""
    H, F, V, S = m.d_model, m.d_ff, m.vocab, m.seq_len
    out = [(0, "tok_emb", (V, H), "emb"), (0, "pos_emb", (S, H), "emb")]
    for layer in range(m.n_layer):
        u = layer + 1
        out += [(u, f"h{layer}.ln1.g", (H,), "one"), (u, f"h{layer}.ln1.b", (H,), "zero"),
                (u, f"h{layer}.w_qkv", (3 * H, H), "w"), (u, f"h{layer}.b_qkv", (3 * H,), "zero"),
                (u, f"h{layer}.w_o", (H, H), "wres"), (u, f"h{layer}.b_o", (H,), "zero"),
                (u, f"h{layer}.ln2.g", (H,), "one"), (u, f"h{layer}.ln2.b", (H,), "zero"),
                (u, f"h{layer}.w_1", (F, H), "w"), (u, f"h{layer}.b_1", (F,), "zero"),
                (u, f"h{layer}.w_2", (H, F), "wres"), (u, f"h{layer}.b_2", (H,), "zero")]
    u = m.n_layer + 1
    out += [(u, "ln_f.g", (H,), "one"), (u, "ln_f.b", (H,), "zero"), (u, "w_head", (V, H), "w")]
    return out


def n_params(m: ModelCfg) -> int:
    return sum(int(np.prod(s)) for _, _, s, _ in param_specs(m))


def round_to_bf16(x: np.ndarray) -> np.ndarray:
    """Round fp32 values to the nearest bf16-representable fp32 (ties to even)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    b = x.view(np.uint32).astype(np.uint64)
    rounding = ((b >> 16) & 1) + 0x7FFF
    r = ((b + rounding) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


def make_params(m: ModelCfg, seed: int = 42) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    std_res = 0.02 / math.sqrt(2 * m.n_layer)
    parts = []
    for _, _, shape, init in param_specs(m):
        n = int(np.prod(shape))
        if init == "one":
            parts.append(np.ones(n, np.float32))
        elif init == "zero":
            parts.append(np.zeros(n, np.float32))
        else:
            std = std_res if init == "wres" else 0.02
            parts.append((rng.standard_normal(n, dtype=np.float32) * np.float32(std)))
    return round_to_bf16(np.concatenate(parts))


def make_tokens(cfg: RunCfg, step: int = 0, zipf: bool = False):
    """(tokens, targets) int32 [M*mb, S]."""
    m = cfg.model
    rng = np.random.Generator(np.random.PCG64(1234 + cfg.index + 1000 * step))
    n = cfg.microbatches * cfg.micro_batch
    S = m.seq_len

    def draw(shape):
        if zipf:
            z = rng.zipf(1.1, size=shape) - 1
            return (z % m.vocab_sample).astype(np.int32)
        return rng.integers(0, m.vocab_sample, size=shape, dtype=np.int64).astype(np.int32)

    if cfg.gpt:
        seq = draw((n, S + 1))
        return np.ascontiguousarray(seq[:, :S]), np.ascontiguousarray(seq[:, 1:])
    return draw((n, S)), draw((n, S))
