"""BASELINE configs[4]: preemption-injection sweep (SURVEY.md §8(d) "C4").

    torchrun --nproc-per-node N tools/sweep_c4.py --config C3 --steps 100 --k 0 1 2 3

For each k: `steps` training steps with k preemptions at steps drawn with
numpy PCG64(seed 7) from [10, 90] (at least 11 steps apart); the victim is
drawn uniformly among the stages (all protected again after the previous
rejoin) and the injection point uniformly over the victim's list; the victim
rejoins (bb_rejoin) 10 steps later. One pipeline serves the whole
sweep (training continues from one k to the next). Reports total samples / total
wall time, the pause of every injection (interrupted step incl. bb_recover
minus the median failure-free step), the failover ("spare tire") step time
and the rejoin time. One JSON line per k on rank 0.
"""
import argparse
import json
import os
import statistics
import sys
import time

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
from synth import get_config, make_params, make_tokens  # noqa: E402


def schedule(k, steps, seed=7):
    rng = np.random.Generator(np.random.PCG64(seed + 100 * k))
    lo, hi = min(10, steps - 1), min(90, steps - 1)
    for _ in range(1000):
        ts = sorted(int(x) for x in rng.integers(lo, hi + 1, size=k))
        if all(b - a >= 11 for a, b in zip(ts, ts[1:])):
            return ts, rng
    raise RuntimeError("cannot place injections")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--k", type=int, nargs="+", default=[0, 1, 2, 3])
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
    # one pipeline for the whole sweep (training simply continues from one k
    # to the next; every k starts and ends on the normal, fully protected plan)
    nid = bench.bcast_bytes(bb.session_id() if rank == 0 else None, ws) if ws > 1 else None
    pipe = bb.Pipeline(m, P, M, micro_batch=mb, rc=True, world_rank=rank, world_size=ws,
                       device=local, session_id=nid,
                       layers_per_stage=bench.device_partition(m, P, -(-P // ws)),
                       frc_retain_bytes=bench.AUTO)   # bench.py's partition and FRC budget
    pipe.load_params(flat)
    pipe.stage_inputs(tok, tgt)
    for _ in range(3):
        pipe.step()
    for k in args.k:
        ts, rng = schedule(k, args.steps)
        plans = {}
        for line in pipe.schedule_dump().splitlines():
            if not line.startswith("#"):
                n = int(line.split()[0])
                plans[n] = plans.get(n, 0) + 1
        normal, fo, pauses, rejoins, injections = [], [], [], [], []
        rejoin_at = {}
        bench.barrier(ws)
        torch.cuda.synchronize()
        t_all = time.perf_counter()
        for t in range(args.steps):
            if t in rejoin_at:
                t0 = time.perf_counter()
                pipe.rejoin()
                rejoins.append(bench.allreduce_max((time.perf_counter() - t0) * 1e3, ws))
            injected = None
            if t in ts:
                v = int(rng.integers(0, P))
                pi = int(rng.integers(0, plans[v] + 1))
                pipe.preempt(v, pi)
                injected = (v, pi)
                rejoin_at[t + 10] = True
            t0 = time.perf_counter()
            status, st = pipe.step()
            if status == "preempted":
                rec = pipe.recover()
                injections.append({"step": t, "victim": injected[0], "at_instr": injected[1],
                                   "brc_mb": rec.brc_mb, "commit": rec.commit})
            dt = bench.allreduce_max((time.perf_counter() - t0) * 1e3, ws)
            if injected:
                pauses.append(dt)
            elif any(t0_ <= t < t0_ + 10 for t0_ in ts):
                fo.append(dt)
            else:
                normal.append(dt)
        bench.barrier(ws)
        wall = time.perf_counter() - t_all
        if any(t0_ + 10 >= args.steps for t0_ in ts):
            pipe.rejoin()                  # back to the normal plan for the next k
        med = statistics.median(normal) if normal else float("nan")
        for inj, p in zip(injections, pauses):
            inj["interrupted_step_ms"] = round(p, 2)
            inj["pause_ms"] = round(p - med, 2)
        if rank == 0:
            print(json.dumps({
                "metric": "C4 preemption sweep: samples/s with k preemptions per 100 steps",
                "config": {"workload": f"{cfg.name} {m.n_layer}L H{m.d_model}, {P} stages on {ws} GPU(s), "
                                       f"M={M}, mb={mb}, EFLB + rejoin after 10 steps",
                           "steps": args.steps, "k": k, "injection_steps": ts},
                "value": round(M * mb * args.steps / wall, 2), "unit": "samples/s",
                "median_step_ms": round(med, 2),
                "failover_step_ms": round(statistics.median(fo), 2) if fo else None,
                "rejoin_ms": [round(r, 2) for r in rejoins],
                "injections": injections}), flush=True)
    pipe.close()
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
