"""Worker for multi-process parity tests; launched by tests/test_gpu_multi.py
through torch.distributed.run. One process per rank; ranks share the visible
GPUs round-robin (rank r on device r % n_gpus), so the cross-process
transport (CUDA IPC + host-shm rendezvous) runs even on a 1-GPU box. Runs a
few steps of a config through the C ABI, optionally injecting a
preemption, and saves each rank's hosted stage states to <out>/rank<r>.npz.
The harness process group is gloo (host-side id broadcast and barriers only;
the library never uses it)."""
import argparse
import dataclasses
import os

# Every node has a main + FRC stream and every NCCL edge its own stream:
# give each its own hardware queue (the default 8 would serialise unrelated
# streams behind spinning P2P kernels). Must precede CUDA initialisation.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2204_12013_b200 as bb  # noqa: E402
from synth import get_config, make_params, make_tokens  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C0")
    ap.add_argument("--prec", default="bf16")
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--victim", type=int, default=-1)
    ap.add_argument("--pi", type=int, default=0)
    ap.add_argument("--stages", type=int, default=0)
    ap.add_argument("--out", required=True)
    ap.add_argument("--rc", default="eflb", help="none / eflb / lflb / efeb")
    ap.add_argument("--events", default="", help="t:v:pi or t:rejoin, comma separated")
    ap.add_argument("--failstop", default="", help="t:v:pi — fail-stop loss armed on v's rank only")
    ap.add_argument("--detect", type=int, default=0, help="bb_opts.detect_ms")
    ap.add_argument("--pipelines", type=int, default=1, help="bb_opts.pipelines (D)")
    a = ap.parse_args()
    rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dev = local % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    cfg = get_config(a.config)
    P = a.stages or cfg.stages
    obj = [bb.session_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    p = bb.Pipeline(cfg.model, P, cfg.microbatches, micro_batch=cfg.micro_batch, rc=a.rc,
                    prec=a.prec, lr=1e-4, world_rank=rank, world_size=ws, device=dev,
                    session_id=obj[0], detect_ms=a.detect, pipelines=a.pipelines)
    p.load_params(make_params(cfg.model))
    losses, rec = [], None
    events = {}
    for e in filter(None, a.events.split(",")):
        f = e.split(":")
        events[int(f[0])] = "rejoin" if f[1] == "rejoin" else (int(f[1]), int(f[2]))
    if a.victim >= 0:
        events[0] = (a.victim, a.pi)
    fs = tuple(int(x) for x in a.failstop.split(":")) if a.failstop else None
    bcfg = dataclasses.replace(cfg, microbatches=a.pipelines * cfg.microbatches)
    for t in range(a.steps):
        tok, tgt = make_tokens(bcfg, t)   # D*M micro-batches
        if fs is not None and fs[0] == t and fs[1] == rank:   # one node per rank
            p.preempt(fs[1], fs[2])
            status, st = p.step(tok, tgt)
            assert status == "preempted"
            p.close()          # waits until the survivors released our memory
            os._exit(0)        # the victim process is gone
        ev = events.get(t)
        if ev == "rejoin":
            p.rejoin()
        elif ev is not None:
            p.preempt(*ev)
        status, st = p.step(tok, tgt)
        loss = st.loss
        if status == "preempted":
            r = p.recover()
            loss, rec = r.loss, r
        losses.append(loss)
        if fs is None:
            dist.barrier()
    out = {"losses": np.array(losses, np.float32), "dump": np.array(p.schedule_dump())}
    if rec is not None:
        out["recovery_dump"] = np.array(p.recovery_dump())
        out["rec"] = np.array([rec.victim, rec.shadow, rec.commit, rec.brc_mb, rec.frc_done_mb,
                               rec.resent_mb, rec.frc_recomputed_mb], np.int64)
        out["rec_loss"] = np.float32(rec.loss)
    for s in range(P * a.pipelines):   # d*P + s: pipeline d's copy
        for what in ("params", "grads", "adam_m", "adam_v"):
            try:
                out[f"{what}_{s}"] = p.read_state(s, what)
            except bb.BambooError:
                pass
    np.savez(os.path.join(a.out, f"rank{rank}.npz"), **out)
    p.close()
    if fs is None:   # gloo cannot barrier over a dead rank
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
