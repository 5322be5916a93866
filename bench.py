"""Benchmark of the Bamboo redundant-computation pipeline step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one process per GPU)

A step = one synchronous 1F1B training step with eager FRC in the bubbles
(BASELINE.json north star) over M*mb synthetic sequences: every stage's
forward/backward, the FRC forward of its successor, P2P activations /
gradients, replica gradient sync and both Adam updates. Workload (default):
BASELINE configs[3] = GPT-2 XL (48 layers, H 1600, 25 heads, S 1024), 8
stages, M=32 micro-batches of 4 sequences — the north-star model. The 8
stages are spread over the N GPUs (N=1: all eight on one B200; N=8: one per
GPU; same model and batch -> strong scaling). At N=1 the FRC retention of
all 8 replicas does not fit next to the 1F1B stash (DESIGN.md §4 "HBM"): the
FRC budget (bb_opts.frc_retain_bytes) keeps what HBM leaves free and
the lazy BRC recomputes the rest. --config C1/C2 select the other models.

Prints ONE JSON line (rank 0). `value` = samples/s with inputs resident in HBM
(bb_stage_inputs), device-timed with CUDA events between synchronised
barriers, max over ranks; `e2e` = the same through bb_step with host buffers
(token upload and loss read-back inside the timed region). Also: RC-off
throughput and the RC overhead, per-node busy / bubble / FRC time, the
recovery matrix (victims 0, 1, P/2, P-1 x first FWD / mid BWD), the GEMM
roofline fraction and the oracle's CPU baseline.
"""
import argparse
import dataclasses
import json
import os

# Every node has a main + FRC stream and every NCCL edge its own stream:
# give each its own hardware queue (the default 8 would serialise unrelated
# streams behind spinning P2P kernels). Must precede CUDA initialisation.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import get_config, make_params, make_tokens  # noqa: E402

MODEL_NAMES = {"C0": "tiny", "C1": "GPT-2 small", "C2": "BERT-large", "C3": "GPT-2 XL"}
BASELINE_METRIC = "samples/sec at 1/2/4/8 B200 with RC vs no-RC; RC overhead %; recovery ms"


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0,
                "fallback": True}


# ------------------------------------------------------------------ clocks
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------- distributed
_HARNESS_DEV = "cuda"   # where the harness's max / sum reductions live


def dist_setup(args):
    global _HARNESS_DEV
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        ngpu = max(1, torch.cuda.device_count())
        if int(os.environ.get("LOCAL_WORLD_SIZE", ws)) > ngpu:
            # more processes than GPUs (a rehearsal of a larger N on a smaller
            # box): ranks share GPUs round-robin and the harness uses gloo,
            # since NCCL refuses two ranks on one device (the library itself
            # never uses NCCL)
            local %= ngpu
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
            _HARNESS_DEV = "cpu"
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        # (the harness's own barriers / max-over-ranks only: the library never uses NCCL)
    return rank, ws, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def allreduce_max(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], device=_HARNESS_DEV)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


def allreduce_sum(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], device=_HARNESS_DEV)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.item()


def bcast_bytes(b, ws):
    if ws == 1:
        return b
    import torch.distributed as dist
    obj = [b]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


# --------------------------------------------------------------- our arm
def timed(pipe, steps, ws, host_inputs=None):
    """Run `steps` steps between synchronised barriers; CUDA events on the
    current stream bracket the region (bb_step synchronises its own streams
    before returning, so the end event follows all of the step's work)."""
    import torch
    barrier(ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches, h2d, d2h = 0, 0, 0
    e0.record()
    for i in range(steps):
        if host_inputs is None:
            status, st = pipe.step()
        else:
            tok, tgt = host_inputs[i % len(host_inputs)]
            status, st = pipe.step(tok, tgt)
        assert status == "ok"
        launches += st.gpu_launches
        h2d += st.h2d_bytes
        d2h += st.d2h_bytes
    e1.record()
    torch.cuda.synchronize()
    barrier(ws)
    ms = allreduce_max(e0.elapsed_time(e1), ws)
    return ms, launches, h2d, d2h


def log(rank, *a):
    if rank == 0:
        print(f"[bench {time.strftime('%H:%M:%S')}]", *a, file=sys.stderr, flush=True)


def balanced_partition(m, P, rc=True, per=1):   # per > 1: exact but slow; see device_partition
    """Blocks per stage (bb_opts.layers_per_stage) that balance the per-node
    work of one micro-batch. An even split by layer count (the default, Q6)
    leaves the last stage with the LM head on top of its blocks: at C1 the
    head's GEMM + cross entropy is ~4 blocks' forward, so the last node
    paces the pipeline. Cost model (per token, FLOP-proportional, calibrated
    on C1 kernel times: block fwd 220 us, bwd 530 us, head + cross entropy
    fwd 900 us, bwd 930 us per micro-batch): block fwd 24H^2 + 4SH (causal:
    halved attention), bwd 2.4x; head fwd 2HV x 0.85, bwd 2HV x 0.87 (the
    head GEMM runs faster per FLOP than a block). A node's
    load is its stage's fwd + bwd plus, with RC, its successor's fwd (FRC).
    Contiguous shards; interior stages keep >= 1 block, the first / last may
    hold only the embedding / the head. With `per` > 1 nodes per GPU
    (contiguous blocks of nodes, the library's default placement) the GPUs
    time-share their nodes, so the objective is the largest per-GPU sum of
    node loads (per = 1: the largest node load)."""
    L, H, S, V = m.n_layer, m.d_model, m.seq_len, m.vocab
    fb = 24.0 * H * H + 4.0 * S * H * (0.5 if m.causal else 1.0)
    bb_ = 2.4 * fb
    fh, bh = 2.0 * H * V * 0.85, 2.0 * H * V * 0.87

    def loads(c):
        f = [c[s] * fb + (fh if s == P - 1 else 0.0) for s in range(P)]
        b = [c[s] * bb_ + (bh if s == P - 1 else 0.0) for s in range(P)]
        return [f[s] + b[s] + (f[(s + 1) % P] if rc and P > 1 else 0.0) for s in range(P)]

    # exact minimax by depth-first search with branch and bound (the load of
    # node s is known once c[s+1] is chosen; the last node's needs c[0])
    A = lambda s, x: x * (fb + bb_) + ((fh + bh) if s == P - 1 else 0.0)   # own fwd + bwd
    F = lambda s, x: (x * fb + (fh if s == P - 1 else 0.0)) if (rc and P > 1) else 0.0
    base, rem = divmod(L, P)
    even = [base + (1 if s >= P - rem else 0) for s in range(P)]
    per = max(1, per)

    def objective(nl):   # node loads -> the largest per-GPU sum
        return max(sum(nl[i:i + per]) for i in range(0, P, per))

    best = [objective(loads(even)), even]

    # depth-first search with branch and bound: node s's load is known once
    # c[s+1] is chosen (the last node's needs c[0]); a GPU's sum once all of
    # its nodes' are. `dev` = the open GPU's partial sum, `cur` = the largest
    # closed one.
    def dfs(c, used, cur, dev):
        s = len(c)
        if max(cur, dev) >= best[0]:
            return
        if s == P:
            if used == L:
                full = max(cur, dev + A(P - 1, c[-1]) + F(0, c[0]))
                if full < best[0] - 1e-9:
                    best[0], best[1] = full, list(c)
            return
        lo = 0 if s in (0, P - 1) else 1
        left = L - used
        need_after = max(0, P - 2 - s) if s < P - 1 else 0   # interior stages still to fill
        for x in range(lo, left - need_after + 1):
            if s == P - 1 and x != left:
                continue
            ncur, ndev = cur, dev
            if s > 0:   # node s-1 is complete now
                ndev = dev + A(s - 1, c[-1]) + F(s, x)
                if s % per == 0:   # ... and so is its GPU
                    ncur, ndev = max(cur, ndev), 0.0
            c.append(x)
            dfs(c, used + x, ncur, ndev)
            c.pop()

    dfs([], 0, 0.0, 0.0)
    return best[1]


def device_partition(m, P, per, alpha=0.8, rc=True):
    """Blocks per stage for `per` nodes per GPU (contiguous node blocks):
    the GPUs time-share their nodes, so the largest per-GPU sum of node loads
    bounds the step, but a pure per-GPU objective piles blocks onto single
    nodes (and the 1F1B critical path runs through every node). Objective:
    max(largest per-GPU sum, alpha * per * largest node load); hill climbing
    by single-block moves from the per-node optimum (balanced_partition).
    Measured at C3 N=4 (profiles/r02_part_*_n4.json): 208.4 samples/s vs
    202.6 for the per-node partition."""
    L, H, S, V = m.n_layer, m.d_model, m.seq_len, m.vocab
    fb = 24.0 * H * H + 4.0 * S * H * (0.5 if m.causal else 1.0)
    bb_ = 2.4 * fb
    fh, bh = 2.0 * H * V * 0.85, 2.0 * H * V * 0.87

    def score(c):
        f = [c[s] * fb + (fh if s == P - 1 else 0.0) for s in range(P)]
        nl = [f[s] + c[s] * bb_ + (bh if s == P - 1 else 0.0) +
              (f[(s + 1) % P] if rc and P > 1 else 0.0) for s in range(P)]
        dev = max(sum(nl[i:i + per]) for i in range(0, P, per))
        return max(dev, alpha * per * max(nl))

    best = balanced_partition(m, P, rc)
    if per <= 1 or per >= P:
        return best
    cur = score(best)
    improved = True
    while improved:
        improved = False
        for i in range(P):
            for j in range(P):
                if i == j or best[i] == 0:
                    continue
                c = list(best)
                c[i] -= 1
                c[j] += 1
                if any(c[k] < 1 for k in range(1, P - 1)):
                    continue
                sc = score(c)
                if sc < cur * (1 - 1e-9):
                    best, cur, improved = c, sc, True
    return best


AUTO = (1 << 64) - 1   # bb_opts.frc_retain_bytes: what HBM leaves free after the rest


def plan_index(pipe, node, kind, nth):
    """Index (into node's current list) just after its nth (1-based) `kind`."""
    idx = [int(f[1]) for f in (l.split() for l in pipe.schedule_dump().splitlines()
                               if not l.startswith("#")) if f[0] == str(node) and f[2] == kind]
    return idx[nth - 1] + 1


def recovery_matrix(pipe, P, M, ws, step_ms, rank):
    """victims {0, 1, P/2, P-1} x {first FWD, ceil(M/2)-th
    BWD}. Per point: the interrupted step + bb_recover (host wall time,
    max over ranks), pause = that - the failure-free step (Q11), one step on
    the failover plan (the spare tire), then bb_rejoin and one normal
    step before the next point."""
    import torch
    out = []
    for v in sorted({0, 1, P // 2, P - 1}):
        for phase, kind, nth in (("first_fwd", "FWD", 1), ("mid_bwd", "BWD", -(-M // 2))):
            pi = plan_index(pipe, v, kind, nth)
            pipe.preempt(v, pi)
            barrier(ws)
            t0 = time.perf_counter()
            status, _ = pipe.step()
            rec = pipe.recover() if status == "preempted" else None
            torch.cuda.synchronize()
            barrier(ws)
            t_int = allreduce_max((time.perf_counter() - t0) * 1e3, ws)
            t1 = time.perf_counter()
            pipe.step()
            barrier(ws)
            t_fo = allreduce_max((time.perf_counter() - t1) * 1e3, ws)
            t2 = time.perf_counter()
            pipe.rejoin()
            barrier(ws)
            t_rj = allreduce_max((time.perf_counter() - t2) * 1e3, ws)
            pipe.step()
            r = {"victim": v, "phase": phase, "at_instr": pi,
                 "interrupted_step_ms": round(t_int, 2), "pause_ms": round(t_int - step_ms, 2),
                 "relative_pause": round((t_int - step_ms) / step_ms, 4),
                 "recover_ms": round(allreduce_max(rec.recover_ms if rec else 0.0, ws), 2),
                 "brc_mb": rec.brc_mb if rec else 0,
                 "frc_reused_mb": rec.frc_done_mb if rec else 0,
                 "frc_recomputed_mb": rec.frc_recomputed_mb if rec else 0,
                 "bytes_resent": int(rec.bytes_resent) if rec else 0,
                 "failover_step_ms": round(t_fo, 2), "rejoin_ms": round(t_rj, 2)}
            log(rank, "recovery", r)
            out.append(r)
    return out


def run_ours(args, rank, ws, local):
    import torch
    import paper_2204_12013_b200 as bb

    cfg = get_config(args.config)
    m = cfg.model
    D = max(1, args.pipelines)   # data-parallel pipelines
    P = max(cfg.stages, -(-ws // D), args.stages)
    M, mb = cfg.microbatches, cfg.micro_batch
    samples = D * M * mb
    def fresh_id():   # every context needs its own rendezvous
        return bcast_bytes(bb.session_id() if rank == 0 else None, ws) if ws > 1 else None
    flat = make_params(m)
    bcfg = dataclasses.replace(cfg, microbatches=D * M)   # all D pipelines' micro-batches
    tok, tgt = make_tokens(bcfg, 0)
    host_batches = [make_tokens(bcfg, s) for s in range(1, 3)]
    per = -(-(D * P) // ws)   # nodes per GPU under the default contiguous placement
    if args.lps:
        lps = [int(x) for x in args.lps.split(",")]
    elif args.partition == "balanced":     # per-node loads
        lps = balanced_partition(m, P)
    elif args.partition == "device":       # per-GPU sums of node loads
        lps = device_partition(m, P, per if D == 1 else 1)
    else:
        lps = None
    common = dict(micro_batch=mb, prec="bf16", world_rank=rank, world_size=ws, device=local,
                  layers_per_stage=lps, pipelines=D)
    e2e_steps = max(1, min(args.steps, args.e2e_steps))

    results = {}
    for rc in (False, True):
        log(rank, f"init rc={rc} P={P} M={M} mb={mb}")
        extra = dict(frc_retain_bytes=AUTO if args.retain == "auto" else int(args.retain),
                     timing=True, frc_persistent=args.frc_persistent) if rc else {}
        pipe = bb.Pipeline(m, P, M, rc=rc, session_id=fresh_id(), **common, **extra)
        pipe.load_params(flat)
        pipe.stage_inputs(tok, tgt)
        for i in range(args.warmup):
            t0 = time.perf_counter()
            _, st = pipe.step()
            log(rank, f"warmup {i}: {1e3 * (time.perf_counter() - t0):.1f} ms host, "
                      f"{st.device_ms:.1f} ms device, loss {st.loss:.4f}, {st.gpu_launches} launches")
        clocks = Clocks(local)
        if rc:
            clocks.start()
        ms, launches, _, _ = timed(pipe, args.steps, ws)
        clk = clocks.stop() if rc else None
        log(rank, f"timed: {ms / args.steps:.2f} ms/step")
        res = dict(ms=ms / args.steps, launches=launches, clocks=clk)
        if rc:
            res["nodes"] = pipe.node_stats()       # the last timed step
            res["retained"] = [pipe.stage_memory(s)[1] for s in range(P)]
            res["slot_mb"] = [round(pipe.stage_memory(s)[0] / 2**20, 1) for s in range(P)]
        # end to end through the public call with host buffers
        ms_e2e, _, h2d, d2h = timed(pipe, e2e_steps, ws, host_inputs=host_batches)
        log(rank, f"e2e: {ms_e2e / e2e_steps:.2f} ms/step")
        pipe.stage_inputs(tok, tgt)
        res.update(e2e_ms=ms_e2e / e2e_steps, h2d=h2d / e2e_steps, d2h=d2h / e2e_steps)
        results[rc] = res
        if rc and args.recovery and D == 1:
            results["recovery"] = recovery_matrix(pipe, P, M, ws, res["ms"], rank)
        pipe.close()
        del pipe
        torch.cuda.empty_cache()

    # Per-kernel device times: the same step (RC on) re-run with every local
    # node on one serialised stream, each kernel bracketed by CUDA events on
    # that stream (concurrent streams would double-count overlapped time).
    log(rank, "profiled (serialised) steps for per-kernel times")
    pipe = bb.Pipeline(m, P, M, rc=True, profile=True, session_id=fresh_id(),
                       frc_retain_bytes=AUTO if args.retain == "auto" else int(args.retain),
                       **common)
    pipe.load_params(flat)
    pipe.stage_inputs(tok, tgt)
    for _ in range(2):
        _, st_prof = pipe.step()
    ks = pipe.kernel_stats()
    prof_step_ms = allreduce_max(st_prof.device_ms, ws)
    pipe.close()
    del pipe
    torch.cuda.empty_cache()

    on, off = results[True], results[False]
    value = samples / (on["ms"] / 1e3)
    pk = peaks()
    gemm_ms = sum(ks[k][1] for k in ks if k.startswith("gemm"))
    gemm_flop = sum(ks[k][2] for k in ks if k.startswith("gemm"))
    gemm_n = sum(ks[k][0] for k in ks if k.startswith("gemm"))
    # profiled totals are per rank over the timed steps; aggregate over ranks
    gemm_ms_all = allreduce_sum(gemm_ms, ws)
    gemm_flop_all = allreduce_sum(gemm_flop, ws)
    achieved = gemm_flop_all / (gemm_ms_all / 1e3) / 1e12 if gemm_ms_all > 0 else 0.0
    launches = allreduce_sum(on["launches"], ws)
    on["h2d"] = allreduce_sum(on["h2d"], ws)
    on["d2h"] = allreduce_sum(on["d2h"], ws)
    recm = results.get("recovery", [])
    if ws > 1:   # every rank's own nodes
        import torch.distributed as dist
        allnodes = [None] * ws
        dist.all_gather_object(allnodes, on["nodes"])
        on["nodes"] = sorted((n for part in allnodes for n in part), key=lambda n: n["node"])
    if rank != 0:
        return
    sust = pk.get("bf16_tflops_sustained", 1377.6)
    roof = {"bound": "tensor", "achieved": round(achieved, 1), "peak": sust, "unit": "TFLOP/s",
            "frac": round(achieved / sust, 4), "traffic": None,
            "kernel": "gemm_tc (tcgen05 bf16, all GEMM launches of the step)",
            "launches_per_step": gemm_n,
            "timing": "CUDA events around every GEMM launch of one full step (RC on), all "
                      "local nodes serialised on one stream; sum of 2MNK over sum of durations",
            "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained (kernel inside a long step)"}
    ncu = os.path.join(ROOT, "profiles", f"r02_ncu_gemm_{cfg.name.lower()}.json")
    if os.path.exists(ncu):
        try:
            d = json.load(open(ncu))
            roof["traffic"] = d.get("dram_bytes_per_launch")
            roof["traffic_source"] = os.path.relpath(ncu, ROOT)
        except Exception:
            pass
    train_flop = useful_flop_per_sample(cfg)
    mid = [r for r in recm if r["phase"] == "mid_bwd" and r["victim"] == P // 2]
    nodes = [{k: (round(v, 2) if isinstance(v, float) else v) for k, v in n.items()}
             for n in on["nodes"]]
    line = {
        "metric": BASELINE_METRIC,
        "value": round(value, 2), "unit": "samples/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(on["ms"], 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded tokens, random-init weights)",
        "config": {"workload": workload_name(cfg, P, D),
                   "stages": P, "microbatches": M, "micro_batch": mb, "global_batch": samples,
                   "seq_len": m.seq_len,
                   "parallelism": (f"dp{D} x " if D > 1 else "") + f"pp{P} on {ws} GPU(s)",
                   "pipelines": D,
                   "layers_per_stage": lps or "even",
                   "frc_retained_per_step": on["retained"], "saved_set_mb": on["slot_mb"],
                   "l2": "working set (weights, stash, FRC retention) >> 126 MB L2"},
        "rc_off": {"value": round(samples / (off["ms"] / 1e3), 2), "ms_per_step": round(off["ms"], 3)},
        "rc_overhead_pct": round(100.0 * (1 - off["ms"] / on["ms"]), 2),
        "rc_slowdown_pct": round(100.0 * (on["ms"] / off["ms"] - 1), 2),
        "recovery_ms": mid[0]["pause_ms"] if mid else None,
        "recovery": recm,
        "nodes": nodes,
        "roofline": roof,
        "model_flops_frac": round(value * train_flop / (ws * pk.get("bf16_tflops", 1657.2) * 1e12), 4),
        "e2e": {"value": round(samples / (on["e2e_ms"] / 1e3), 2), "unit": "samples/s",
                "h2d_bytes_per_step": int(on["h2d"]), "d2h_bytes_per_step": int(on["d2h"]),
                "steps": e2e_steps},
        "gpu_launches": int(launches),
        "clocks": on["clocks"],
        "kernel_ms_per_step": {k: round(v[1], 3) for k, v in ks.items()},
        "serialised_step_ms": round(prof_step_ms, 2),
    }
    if args.cpu_baseline and ws == 1:   # the oracle leg runs on rank 0 at N=1 only
        log(rank, "cpu baseline (oracle)")
        line["cpu_baseline"] = cpu_baseline(cfg, budget_s=args.cpu_budget)
    print(json.dumps(line), flush=True)


def useful_flop_per_sample(cfg):
    """3 x forward FLOPs per sample: GEMMs + causal attention
    counted as half, LM head included."""
    m = cfg.model
    H, F, V, S = m.d_model, m.d_ff, m.vocab, m.seq_len
    per_tok = m.n_layer * (2 * (3 * H * H + H * H + 2 * H * F)) + 2 * H * V
    attn = m.n_layer * 2 * 2 * S * H * (0.5 if m.causal else 1.0)
    return 3 * S * (per_tok + attn)


# ------------------------------------------------ oracle (CPU) baseline leg
def cpu_baseline(cfg, budget_s=20.0):
    """Time the fp64 oracle as it stands on this host: one sequence through
    one transformer block and through the LM head at the config's width,
    forward + backward, then scale to the full step with RC (12 blocks fwd +
    bwd + head, plus the FRC forward of every stage = one more forward)."""
    import threadpoolctl
    from oracle import model as om
    m = cfg.model
    lay = om.Layout(m)
    flat = make_params(m).astype(np.float64)
    th = lay.tensors(flat, 0, lay.total)
    gr = lay.tensors(np.zeros(lay.total), 0, lay.total)
    tok, tgt = make_tokens(cfg, 0)
    tok, tgt = tok[:1], tgt[:1]
    ntok = tok.size
    x = om.embedding_fwd(th["tok_emb"], th["pos_emb"], tok)
    t_fb, t_f, t_hf, t_hb, reps = 0.0, 0.0, 0.0, 0.0, 0
    t_start = time.perf_counter()
    while reps == 0 or time.perf_counter() - t_start < budget_s / 2:
        t0 = time.perf_counter()
        y, sv = om.unit_fwd(lay, 1, th, x, tok, tgt, ntok)
        t1 = time.perf_counter()
        om.unit_bwd(lay, 1, th, gr, sv, np.ones_like(y), tok, tgt, ntok)
        t2 = time.perf_counter()
        loss, svh = om.unit_fwd(lay, m.n_layer + 1, th, x, tok, tgt, ntok)
        t3 = time.perf_counter()
        om.unit_bwd(lay, m.n_layer + 1, th, gr, svh, None, tok, tgt, ntok)
        t4 = time.perf_counter()
        t_f += t1 - t0
        t_fb += t2 - t0
        t_hf += t3 - t2
        t_hb += t4 - t3
        reps += 1
    per_seq = (m.n_layer * (t_fb + t_f) + (t_hf + t_hb) + t_hf) / reps
    info = threadpoolctl.threadpool_info()
    threads = max([i.get("num_threads", 1) for i in info] or [1])
    return {"value": round(1.0 / per_seq, 5), "unit": "samples/s", "cores": threads,
            "host_cpus": os.cpu_count(), "kind": "oracle (extrapolated)",
            "sample": f"{reps} reps of 1 sequence (S={m.seq_len}) through 1 block + LM head at "
                      f"{cfg.name} width, fp64 numpy fwd+bwd, scaled to {m.n_layer} blocks fwd+bwd"
                      f" + head + FRC forward"}


def workload_name(cfg, P, D=1):
    """config.workload of a bench line (both arms use the same string)."""
    m = cfg.model
    return (f"{cfg.name}: {MODEL_NAMES.get(cfg.name, cfg.name)} {m.n_layer}L H{m.d_model} "
            f"S{m.seq_len} {'causal' if m.causal else 'bidirectional'}, {P} stages, "
            f"M={cfg.microbatches}, mb={cfg.micro_batch}, EFLB (eager FRC, lazy BRC)"
            + (f", {D} data-parallel pipelines" if D > 1 else ""))


def run_reference(args, rank, ws):
    if rank != 0:
        return
    cfg = get_config(args.config)
    budget = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        cpu_baseline(cfg, budget_s=budget)
    vals = []
    t0 = time.perf_counter()
    last = None
    for _ in range(args.steps):
        last = cpu_baseline(cfg, budget_s=budget)
        vals.append(last["value"])
    wall = time.perf_counter() - t0
    v = statistics.median(vals)
    line = {"metric": BASELINE_METRIC, "impl": "reference", "value": v, "unit": "samples/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * wall / args.steps, 1), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded tokens, random-init weights)",
            # our arm's workload (the oracle times a bounded sample of it: cpu_baseline)
            "config": {"workload": workload_name(cfg, max(cfg.stages, ws, args.stages),
                                                 max(1, args.pipelines)),
                       "stages": max(cfg.stages, ws, args.stages),
                       "microbatches": cfg.microbatches, "micro_batch": cfg.micro_batch,
                       "global_batch": max(1, args.pipelines) * cfg.microbatches * cfg.micro_batch,
                       "seq_len": cfg.model.seq_len, "implementation": "fp64 oracle on the host"},
            "cpu_baseline": dict(last, value=v),
            "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3",
                    help="C3 (GPT-2 XL, the north-star model) by default; C1 / C2 / C0")
    ap.add_argument("--stages", type=int, default=0,
                    help="pipeline stages (default: the config's, at least N)")
    ap.add_argument("--lps", default="", help="explicit layers_per_stage, comma separated")
    ap.add_argument("--partition", default="device", choices=["balanced", "device", "even"],
                    help="blocks per stage: cost-balanced per GPU (default; = per node when "
                         "each GPU has one node or all of them), per node, or even by count (Q6)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--e2e-steps", type=int, default=5,
                    help="steps of the end-to-end (host buffers) measurement")
    ap.add_argument("--retain", default="auto",
                    help="frc_retain_bytes per node: auto (free HBM) or bytes (0 = all M)")
    ap.add_argument("--no-recovery", dest="recovery", action="store_false")
    ap.add_argument("--frc-persistent", action="store_true",
                    help="FRC GEMMs on persistent full-device grids (bb_opts.frc_persistent) "
                         "instead of one CTA per tile")
    ap.add_argument("--pipelines", type=int, default=1,
                    help="D data-parallel pipelines (bb_opts.pipelines; the recovery matrix "
                         "runs only at D=1)")
    args = ap.parse_args()
    if args.impl == "reference":
        # the oracle arm needs no GPU and no process group: rank 0 runs it,
        # the other ranks exit 0 at once
        run_reference(args, int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")))
        return
    rank, ws, local = dist_setup(args)
    run_ours(args, rank, ws, local)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
