"""Host logic of bench.py (no GPU): the stage partitions it passes as
bb_opts.layers_per_stage. balanced_partition must be the exact minimax of
the per-node load model (checked by brute force over every contiguous split
of small models); device_partition must never be worse than it on its own
objective (largest per-GPU sum, node maximum kept in check) and must fall
back to it with one node per GPU or all nodes on one GPU."""
import dataclasses
import itertools
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from synth import get_config  # noqa: E402


def _loads(m, c, rc=True):
    P = len(c)
    H, S, V = m.d_model, m.seq_len, m.vocab
    fb = 24.0 * H * H + 4.0 * S * H * (0.5 if m.causal else 1.0)
    bb_ = 2.4 * fb
    fh, bh = 2.0 * H * V * 0.85, 2.0 * H * V * 0.87
    f = [c[s] * fb + (fh if s == P - 1 else 0.0) for s in range(P)]
    return [f[s] + c[s] * bb_ + (bh if s == P - 1 else 0.0) + (f[(s + 1) % P] if rc else 0.0)
            for s in range(P)]


def _splits(L, P):
    """Every contiguous split: interior stages >= 1 block, ends >= 0."""
    for cuts in itertools.product(range(L + 1), repeat=P - 1):
        c = [cuts[0]] + [cuts[i] - cuts[i - 1] for i in range(1, P - 1)] + [L - cuts[-1]]
        if min(c) < 0 or any(x < 1 for x in c[1:-1]):
            continue
        yield c


def test_balanced_partition_is_the_exact_minimax():
    base = get_config("C1").model
    for L, P in ((6, 3), (8, 4), (9, 3), (7, 4)):
        m = dataclasses.replace(base, n_layer=L)
        best = min(max(_loads(m, c)) for c in _splits(L, P))
        got = bench.balanced_partition(m, P)
        assert sum(got) == L and len(got) == P
        assert abs(max(_loads(m, got)) - best) <= 1e-9 * best, (L, P, got)


def test_device_partition_objective_and_fallbacks():
    for name in ("C1", "C2"):   # (C3: same code path, ~10 s per search)
        m = get_config(name).model
        P = 8
        node = bench.balanced_partition(m, P)
        assert bench.device_partition(m, P, 1) == node      # one node per GPU
        assert bench.device_partition(m, P, P) == node      # all nodes on one GPU
        for per in (2, 4):
            dev = bench.device_partition(m, P, per)
            assert sum(dev) == m.n_layer and all(x >= 1 for x in dev[1:-1])

            def obj(c):
                nl = _loads(m, c)
                return max(max(sum(nl[i:i + per]) for i in range(0, P, per)),
                           0.8 * per * max(nl))
            assert obj(dev) <= obj(node) * (1 + 1e-12), (name, per, dev, node)
