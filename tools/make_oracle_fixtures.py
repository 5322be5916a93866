"""Write the oracle fixtures of the PT1 / PT2 parity tiers (SURVEY.md §8(c)
"Oracle cost"): one Adam step of the plain definition (oracle.model.train_step,
O2 brute force, fp64) at full model width on seeded synthetic inputs, stored
as per-tensor summaries plus sampled elements, so the GPU tests can check the
full-width paths without running a multi-minute fp64 step on the GPU box.

Calls only oracle/ and synth/ (the stored values never come from the CUDA
path). Per tensor: max|ref| of the gradient, Adam m, v and the parameter
update, the Frobenius norm of the gradient, and SAMPLE seeded indices
(including the argmax of |g|) with the gradient, m, v and post-Adam value
there.

    python tools/make_oracle_fixtures.py [name ...]   (names: see CASES)
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import model as om  # noqa: E402
from synth import depth_reduced, get_config, make_params, make_tokens  # noqa: E402
import dataclasses  # noqa: E402

LR, B1, B2, EPS = 1e-4, 0.9, 0.999, 1e-8
SAMPLE = 256


def cases():
    c1 = get_config("C1")
    return {
        # PT1: the whole C1 model (12 layers, 4 stages, S=1024, V=50304) on
        # 8 micro-batches of 1 sequence (the named batch has 8 of 8: 1/8 of it)
        "pt1_c1": dataclasses.replace(c1, micro_batch=1),
        # PT2: C2 / C3 width (H, heads, F, S, V, P), one block per stage
        "pt2_c2": depth_reduced("C2", 1, 4, 1),
        "pt2_c3": depth_reduced("C3", 1, 4, 1),
    }


def summarise(lay, g, p0, p1, m1, v1, seed):
    rng = np.random.default_rng(seed)
    out = {}
    for _, name, shape, off in lay.entries:
        n = int(np.prod(shape))
        sl = slice(off, off + n)
        gi = g[sl]
        idx = np.unique(np.concatenate([rng.integers(0, n, SAMPLE), [int(np.argmax(np.abs(gi)))]]))
        out[name] = dict(
            idx=idx.astype(np.int64), g=gi[idx], m=m1[sl][idx], v=v1[sl][idx], p=p1[sl][idx],
            p0=p0[sl][idx], gmax=np.abs(gi).max(), gnorm=np.linalg.norm(gi),
            mmax=np.abs(m1[sl]).max(), vmax=np.abs(v1[sl]).max(),
            umax=np.abs(p1[sl] - p0[sl]).max())
    return out


def make(name, cfg):
    lay = om.Layout(cfg.model)
    flat = make_params(cfg.model).astype(np.float64)
    tok, tgt = make_tokens(cfg, 0)
    t0 = time.time()
    z = np.zeros(lay.total)
    loss, g, p1, m1, v1 = om.train_step(lay, flat, z, z.copy(), 1, tok, tgt, LR, B1, B2, EPS)
    dt = time.time() - t0
    summ = summarise(lay, g, flat, p1, m1, v1, seed=11)
    arrs = {"loss": np.float64(loss), "oracle_s": np.float64(dt)}
    for tname, d in summ.items():
        for key, val in d.items():
            arrs[f"{tname}|{key}"] = np.asarray(val)
    path = os.path.join(ROOT, "tests", "golden", f"{name}.npz")
    np.savez_compressed(path, **arrs)
    print(f"{name}: loss {loss:.6f}, {dt:.0f} s -> {path}", flush=True)


if __name__ == "__main__":
    want = sys.argv[1:] or list(cases())
    for n in want:
        make(n, cases()[n])
