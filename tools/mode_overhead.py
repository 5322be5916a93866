"""RC modes side by side (PAPER tab:time-overhead P:874-886 and
fig:pause P:908-912): per-step time of NONE / LFLB / EFLB / EFEB on the same
workload, the overhead of each against NONE, and the pause of a preemption of
the middle node at its ceil(M/2)-th backward - Q11: interrupted step
including bb_recover minus the failure-free step. One JSON line (rank 0).

    python tools/mode_overhead.py [--config C1] [--steps 5] [--warmup 2]
    torchrun --nproc-per-node N tools/mode_overhead.py --config C3 ...
"""
import argparse
import json
import os
import sys
import time

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from synth import get_config, make_params, make_tokens  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C1")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--modes", nargs="+", default=["none", "lflb", "eflb", "efeb"])
    args = ap.parse_args()
    rank, ws, local = bench.dist_setup(args)
    import torch
    import paper_2204_12013_b200 as bb
    cfg = get_config(args.config)
    m = cfg.model
    P = max(cfg.stages, ws)
    M, mb = cfg.microbatches, cfg.micro_batch
    flat = make_params(m)
    tok, tgt = make_tokens(cfg, 0)
    lps = bench.device_partition(m, P, -(-P // ws))   # bench.py's default partition
    out = {"config": f"{cfg.name}, {P} stages on {ws} GPU(s), M={M}, mb={mb}", "modes": {}}
    for mode in args.modes:
        sid = bench.bcast_bytes(bb.session_id() if rank == 0 else None, ws) if ws > 1 else None
        pipe = bb.Pipeline(m, P, M, micro_batch=mb, rc=mode, world_rank=rank, world_size=ws,
                           device=local, session_id=sid, layers_per_stage=lps,
                           frc_retain_bytes=bench.AUTO if mode in ("eflb", "efeb") else 0)
        pipe.load_params(flat)
        pipe.stage_inputs(tok, tgt)
        for _ in range(args.warmup):
            pipe.step()
        ms, _, _, _ = bench.timed(pipe, args.steps, ws)
        step_ms = ms / args.steps
        r = {"step_ms": round(step_ms, 2), "samples_per_s": round(M * mb / (step_ms / 1e3), 2)}
        if mode != "none":
            v = P // 2
            pi = bench.plan_index(pipe, v, "BWD", -(-M // 2))
            pipe.preempt(v, pi)
            bench.barrier(ws)
            t0 = time.perf_counter()
            status, _ = pipe.step()
            rec = pipe.recover() if status == "preempted" else None
            torch.cuda.synchronize()
            bench.barrier(ws)
            t_int = bench.allreduce_max((time.perf_counter() - t0) * 1e3, ws)
            r.update(pause_ms=round(t_int - step_ms, 2),
                     relative_pause=round((t_int - step_ms) / step_ms, 4),
                     brc_mb=rec.brc_mb if rec else None,
                     frc_recomputed_mb=rec.frc_recomputed_mb if rec else None)
        out["modes"][mode] = r
        bench.log(rank, mode, r)
        pipe.close()
        del pipe
        torch.cuda.empty_cache()
    base = out["modes"].get("none", {}).get("step_ms")
    if base:
        for mode, r in out["modes"].items():
            r["overhead_pct"] = round(100.0 * (r["step_ms"] / base - 1), 2)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
