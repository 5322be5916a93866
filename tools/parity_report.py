"""Per-tensor max-normwise parity table (tests/parity.py metric) of the GPU
path against the fp64 oracle: gradients of one step for several seeded input
batches of C0 and a 3-stage bidirectional C0 variant, bf16 and fp32. Writes
JSON (tensor -> worst error over the batches) to argv[1] or stdout."""
import dataclasses
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import paper_2204_12013_b200 as bb  # noqa: E402
from oracle import pipeline as opipe  # noqa: E402
from parity import normwise, tensor_slices  # noqa: E402
from synth import get_config, make_params, make_tokens  # noqa: E402


def cases():
    c0 = get_config("C0")
    bid = dataclasses.replace(c0, model=dataclasses.replace(c0.model, causal=False, n_layer=5),
                              stages=3, microbatches=5, gpt=False)
    return {"C0": c0, "C0-bidir-3stage": bid}


def run(cfg, prec, batches):
    flat = make_params(cfg.model)
    worst = {}
    for t in batches:
        tok, tgt = make_tokens(cfg, t)
        ref = opipe.Pipeline(cfg, flat, rc=True)
        _, rl = ref.step(tok, tgt)
        rg = ref.full_grads()
        p = bb.Pipeline(cfg.model, cfg.stages, cfg.microbatches, micro_batch=cfg.micro_batch,
                        prec=prec)
        p.load_params(flat)
        _, st = p.step(tok, tgt)
        g = np.concatenate([p.read_state(s, "grads") for s in range(cfg.stages)])
        p.close()
        worst["loss"] = max(worst.get("loss", 0.0), abs(st.loss - rl) / abs(rl))
        for n, a, b in tensor_slices(ref.lay, 0, ref.lay.total):
            worst[n] = max(worst.get(n, 0.0), normwise(g[a:b], rg[a:b]))
    return dict(sorted(worst.items(), key=lambda kv: -kv[1]))


if __name__ == "__main__":
    out = {}
    for name, cfg in cases().items():
        for prec in ("bf16", "fp32"):
            out[f"{name}/{prec}"] = run(cfg, prec, range(6) if prec == "bf16" else range(2))
            top = list(out[f"{name}/{prec}"].items())[:6]
            print(name, prec, [(k, f"{v:.2e}") for k, v in top], flush=True)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            json.dump(out, f, indent=1)
