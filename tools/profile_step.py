"""One warm-up + one profiled step of a config on cuda:0 (for ncu launch lists)."""
import argparse, os, sys

# Every node has a main + FRC stream and every NCCL edge its own stream:
# give each its own hardware queue (the default 8 would serialise unrelated
# streams behind spinning P2P kernels). Must precede CUDA initialisation.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_12013_b200 as bb
from synth import get_config, make_params, make_tokens

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C1")
ap.add_argument("--rc", type=int, default=1)
ap.add_argument("--steps", type=int, default=2)
a = ap.parse_args()
cfg = get_config(a.config)
p = bb.Pipeline(cfg.model, cfg.stages, cfg.microbatches, micro_batch=cfg.micro_batch, rc=bool(a.rc))
p.load_params(make_params(cfg.model))
tok, tgt = make_tokens(cfg, 0)
p.stage_inputs(tok, tgt)
for i in range(a.steps):
    _, st = p.step()
    print(f"step {i}: {st.device_ms:.1f} ms, loss {st.loss:.4f}, {st.gpu_launches} launches", flush=True)
p.close()
