"""Warm-up + profiled steps of a config on cuda:0, with bench.py's stage
partition and FRC budget (for ncu launch lists and ncu --set full captures).

    python tools/profile_step.py [--config C3] [--rc eflb|none] [--steps 2]
"""
import argparse
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2204_12013_b200 as bb  # noqa: E402
from synth import get_config, make_params, make_tokens  # noqa: E402
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--rc", default="eflb")
ap.add_argument("--steps", type=int, default=2)
a = ap.parse_args()
cfg = get_config(a.config)
m = cfg.model
rc = a.rc != "none"
p = bb.Pipeline(m, cfg.stages, cfg.microbatches, micro_batch=cfg.micro_batch, rc=a.rc,
                layers_per_stage=bench.balanced_partition(m, cfg.stages, rc),
                frc_retain_bytes=bench.AUTO if rc else 0)
p.load_params(make_params(m))
tok, tgt = make_tokens(cfg, 0)
p.stage_inputs(tok, tgt)
for i in range(a.steps):
    _, st = p.step()
    print(f"step {i}: {st.device_ms:.1f} ms, loss {st.loss:.4f}, {st.gpu_launches} launches",
          flush=True)
p.close()
