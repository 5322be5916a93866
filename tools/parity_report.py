"""Per-tensor parity report of one C0 step (GPU vs fp64 oracle)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2204_12013_b200 as bb
from oracle import pipeline as opipe
from synth import get_config, make_params, make_tokens
from parity import tensor_slices, normwise

name = sys.argv[1] if len(sys.argv) > 1 else "C0"
cfg = get_config(name)
flat = make_params(cfg.model)
tok, tgt = make_tokens(cfg, 0)
ref = opipe.Pipeline(cfg, flat, rc=True)
_, rl = ref.step(tok, tgt)
rg = ref.full_grads()
for prec in ("bf16", "fp32"):
    p = bb.Pipeline(cfg.model, cfg.stages, cfg.microbatches, micro_batch=cfg.micro_batch, prec=prec)
    p.load_params(flat)
    _, st = p.step(tok, tgt)
    g = np.concatenate([p.read_state(s, "grads") for s in range(cfg.stages)])
    errs = sorted(((normwise(g[a:b], rg[a:b]), n) for n, a, b in tensor_slices(ref.lay, 0, ref.lay.total)), reverse=True)
    print(prec, "loss rel", abs(st.loss - rl) / abs(rl), "worst grads:", [(f"{e:.2e}", n) for e, n in errs[:8]])
    print(prec, "median", np.median([e for e, _ in errs]))
    p.close()
