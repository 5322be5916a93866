"""FRC retention tiers side by side ("swap out these data to CPU memory";
SURVEY Q10, §8(f)-4): the same EFLB workload with the FRC saved sets
beyond a small HBM budget (a) recomputed by the lazy BRC (the default) or
(b) swapped to pinned host memory and copied back by the BRC, against (c)
the automatic HBM budget. Per-step time and the pause of a preemption of the
middle node at its ceil(M/2)-th backward. One JSON line (rank 0).

    torchrun --nproc-per-node N tools/swap_cost.py --config C3 [--keep 4]
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
    ap.add_argument("--config", default="C3")
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--keep", type=int, default=4, help="saved sets kept in HBM per replica")
    ap.add_argument("--swap-sets", type=int, default=0,
                    help="saved sets per replica in pinned host memory (0 = all the rest)")
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
    lps = bench.balanced_partition(m, P)
    probe = bb.Pipeline(m, P, M, micro_batch=mb, rc="eflb", world_rank=rank, world_size=ws,
                        device=local, layers_per_stage=lps, frc_retain_bytes=1,
                        session_id=bench.bcast_bytes(bb.session_id() if rank == 0 else None, ws)
                        if ws > 1 else None)
    slot = max(probe.stage_memory(s)[0] for s in range(P))
    probe.close()
    del probe
    torch.cuda.empty_cache()
    variants = {"hbm_auto": dict(frc_retain_bytes=bench.AUTO),
                "recompute": dict(frc_retain_bytes=args.keep * slot),
                "host_swap": dict(frc_retain_bytes=args.keep * slot,
                                  frc_swap_bytes=(args.swap_sets or M - args.keep) * slot)}
    out = {"config": f"{cfg.name}, {P} stages on {ws} GPU(s), M={M}, mb={mb}, EFLB",
           "saved_set_mb": round(slot / 2**20, 1), "keep_in_hbm": args.keep,
           "swap_sets": args.swap_sets or M - args.keep, "variants": {}}
    for name, kw in variants.items():
        sid = bench.bcast_bytes(bb.session_id() if rank == 0 else None, ws) if ws > 1 else None
        pipe = bb.Pipeline(m, P, M, micro_batch=mb, rc="eflb", world_rank=rank, world_size=ws,
                           device=local, session_id=sid, layers_per_stage=lps, **kw)
        pipe.load_params(flat)
        pipe.stage_inputs(tok, tgt)
        for _ in range(args.warmup):
            pipe.step()
        ms, _, _, _ = bench.timed(pipe, args.steps, ws)
        step_ms = ms / args.steps
        r = {"step_ms": round(step_ms, 2), "samples_per_s": round(M * mb / (step_ms / 1e3), 2),
             "retained": [pipe.stage_memory(s)[1] for s in range(P)]}
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
                 frc_recomputed_mb=rec.frc_recomputed_mb if rec else None,
                 frc_swapped_mb=rec.frc_swapped_mb if rec else None)
        out["variants"][name] = r
        bench.log(rank, name, r)
        pipe.close()
        del pipe
        torch.cuda.empty_cache()
    if rank == 0:
        print(json.dumps(out), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
