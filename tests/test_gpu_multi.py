"""Multi-process parity (one process per rank; the library's CUDA-IPC
transport between ranks, rendezvous in host shared memory): the pipeline
spread over 2 (or 4) processes must give exactly the single-process results
(same kernels, same order => bit-identical) and recover from an injected
preemption bit-identically. Ranks share the visible GPUs round-robin, so on
a 1-GPU box every rank runs on cuda:0 and the cross-process path (IPC
memory + interprocess events between processes) is still exercised; on a
multi-GPU box the copies cross NVLink."""
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

from oracle import pipeline as opipe, plan as opl
from synth import get_config, make_params, make_tokens

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ngpus():
    import torch
    return torch.cuda.device_count()


def run_mp(n, **kw):
    d = tempfile.mkdtemp()
    args = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
            "--master-addr=127.0.0.1", f"--master-port={29500 + os.getpid() % 1000}",
            os.path.join(ROOT, "tests", "mp_worker.py"), "--out", d]
    for k, v in kw.items():
        args += [f"--{k}", str(v)]
    r = subprocess.run(args, capture_output=True, text=True, timeout=240)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return [dict(np.load(os.path.join(d, f"rank{i}.npz"))) if
            os.path.exists(os.path.join(d, f"rank{i}.npz")) else None for i in range(n)]


def merged(ranks, P, what):
    out = []
    for s in range(P):
        got = [r[f"{what}_{s}"] for r in ranks if f"{what}_{s}" in r]
        assert got, (what, s)
        out.append(got[0])
    return np.concatenate(out)


def single(cfg, steps, victim=-1, pi=0):
    import paper_2204_12013_b200 as bb
    p = bb.Pipeline(cfg.model, cfg.stages, cfg.microbatches, micro_batch=cfg.micro_batch, rc=True,
                    lr=1e-4)
    p.load_params(make_params(cfg.model))
    losses = []
    for t in range(steps):
        tok, tgt = make_tokens(cfg, t)
        if t == 0 and victim >= 0:
            p.preempt(victim, pi)
        status, st = p.step(tok, tgt)
        losses.append(p.recover().loss if status == "preempted" else st.loss)
    state = {w: np.concatenate([p.read_state(s, w) for s in range(cfg.stages)])
             for w in ("params", "grads", "adam_m", "adam_v")}
    p.close()
    return losses, state


@pytest.mark.parametrize("n,P", [(2, 2), (2, 4), (4, 4)])
def test_multi_gpu_equals_single_process(n, P):
    """P stages over n GPUs (n < P: several nodes per process, device-local
    edges next to NCCL ones) == all P stages in one process, bit for bit."""
    import dataclasses
    c = dataclasses.replace(get_config("C0"), stages=P)
    ranks = run_mp(n, config="C0", stages=P, steps=2)
    losses, state = single(c, 2)
    assert [float(x) for x in ranks[-1]["losses"]] == [float(x) for x in losses]
    for w in state:
        assert np.array_equal(merged(ranks, P, w), state[w]), w
    per = -(-P // n)
    want = opl.dump(P, c.microbatches, True, opl.partition(4, P),
                    opl.normal_plans(P, c.microbatches, True),
                    device={i: min(i // per, n - 1) for i in range(P)})
    assert str(ranks[0]["dump"]) == want


@pytest.mark.parametrize("victim,pi", [(1, 9), (0, 5), (1, 0), (0, 24)])
def test_multi_gpu_recovery_bitwise(victim, pi):
    cfg = get_config("C0")
    ranks = run_mp(2, config="C0", steps=2, victim=victim, pi=pi)
    losses, state = single(cfg, 2)   # failure-free reference
    survivor = ranks[(victim - 1) % 2]
    assert [float(x) for x in survivor["losses"]] == [float(x) for x in losses]
    assert str(survivor["recovery_dump"]) == opl.recovery_dump(2, cfg.microbatches, victim, pi)
    for w in state:
        assert np.array_equal(merged([survivor], 2, w), state[w]), w


def test_multi_gpu_rejoin_sequence_bitwise():
    """Two ranks, four nodes: preempt node 2 (cross-rank shadow), rejoin, then
    preempt node 1, rejoin: every step equals the failure-free single-process
    run bit for bit."""
    import dataclasses
    c = dataclasses.replace(get_config("C0"), stages=4)
    ranks = run_mp(2, config="C0", stages=4, steps=6, events="0:2:13,2:rejoin,3:1:20,5:rejoin")
    losses, state = single(c, 6)
    assert [float(x) for x in ranks[-1]["losses"]] == [float(x) for x in losses]
    for w in state:
        assert np.array_equal(merged(ranks, 4, w), state[w]), w


@pytest.mark.parametrize("n,victim,pi", [(2, 1, 9), (4, 2, 13), (4, 0, 7), (4, 3, 16)])
def test_failstop_detection_and_recovery_bitwise(n, victim, pi):
    """Fail-stop mode (bb_opts.detect_ms): bb_preempt is called on
    the victim's rank ONLY; that process stops at instruction pi, goes silent
    and exits. The survivors notice the stopped heartbeat after detect_ms,
    run to quiescence, agree on the cut from the messages the victim had
    delivered, recover without it, and keep training: the survivors' state
    after the interrupted step and two failover steps equals the failure-free
    single-process run bit for bit."""
    import dataclasses
    c = dataclasses.replace(get_config("C0"), stages=n)
    ranks = run_mp(n, config="C0", stages=n, steps=3, failstop=f"1:{victim}:{pi}", detect=300)
    assert ranks[victim] is None                      # the victim left no output
    losses, state = single(c, 3)
    live = [r for r in ranks if r is not None]
    for t in range(3):   # whichever survivor hosted the last stage at step t
        if t == 0 and victim == n - 1:
            continue          # step 0 ran before the loss: its loss left with the victim
        got = [float(r["losses"][t]) for r in live if not np.isnan(r["losses"][t])]
        assert got and all(g == float(losses[t]) for g in got), (
            t, got, losses[t], [(r.get("rec"), r["losses"], str(r.get("recovery_dump", ""))[:3000])
                                for r in live])
    for w in state:
        assert np.array_equal(merged(live, n, w), state[w]), w


@pytest.mark.parametrize("mode", ["efeb", "lflb"])
def test_multi_process_modes_bitwise(mode):
    """EFEB's duplicate gradients (node s -> s-2) and LFLB cross process
    boundaries (3 ranks, one node each): a failure-free step and an injected
    preemption of node 1 both equal the single-process failure-free run."""
    import dataclasses
    c = dataclasses.replace(get_config("C0"), stages=3)
    losses, state = single(c, 2)
    for extra in ({}, {"victim": 1, "pi": 12}):
        ranks = run_mp(3, config="C0", stages=3, steps=2, rc=mode, **extra)
        for t in range(2):
            got = [float(r["losses"][t]) for r in ranks if not np.isnan(r["losses"][t])]
            assert got and all(g == float(losses[t]) for g in got), (mode, extra, t)
        for w in state:
            assert np.array_equal(merged(ranks, 3, w), state[w]), (mode, extra, w)


def single_dp(cfg, D, steps, rc="eflb"):
    """D pipelines in one process, failure-free: per-step losses and every
    pipeline's copy of every stage (index d*P + s)."""
    import dataclasses
    import paper_2204_12013_b200 as bb
    p = bb.Pipeline(cfg.model, cfg.stages, cfg.microbatches, micro_batch=cfg.micro_batch, rc=rc,
                    lr=1e-4, pipelines=D)
    p.load_params(make_params(cfg.model))
    bcfg = dataclasses.replace(cfg, microbatches=D * cfg.microbatches)
    losses = []
    for t in range(steps):
        status, st = p.step(*make_tokens(bcfg, t))
        losses.append(st.loss)
    G = D * cfg.stages
    state = {w: np.concatenate([p.read_state(g, w) for g in range(G)])
             for w in ("params", "grads", "adam_m", "adam_v")}
    p.close()
    return losses, state


@pytest.mark.parametrize("n,victim,pi", [(4, -1, 0), (2, -1, 0), (4, 3, 12), (4, 0, 22),
                                         (2, 1, 25)])
def test_multi_process_dp_bitwise(n, victim, pi):
    """D=2 pipelines of P=2 (4 nodes) over n processes: n=4 puts every edge
    (activations, gradients, replica sync, all-reduce) across processes;
    n=2 gives each process one pipeline, so only the all-reduce crosses. The
    per-rank loss shares add up to the single-process loss and every
    pipeline's state equals the single-process D=2 run bit for bit, also
    after a preemption (the other pipeline's all-reduce waits for the
    victim's shadow, which replays it)."""
    cfg = get_config("C0")
    D, P = 2, cfg.stages
    losses, state = single_dp(cfg, D, 2)
    extra = {"victim": victim, "pi": pi} if victim >= 0 else {}
    ranks = run_mp(n, config="C0", stages=P, steps=2, pipelines=D, **extra)
    for t in range(2):
        parts = [np.float32(r["losses"][t]) for r in ranks if not np.isnan(r["losses"][t])]
        assert len(parts) == D, parts   # one share per pipeline, on its last stage's rank
        tot = np.float32(0)
        for x in parts:
            tot = np.float32(tot + x)
        assert tot == np.float32(losses[t]), (t, parts, losses[t])
    for w in state:
        assert np.array_equal(merged(ranks, D * P, w), state[w]), w


@pytest.mark.parametrize("victim,pi", [(1, 12), (2, 22), (3, 5)])
def test_failstop_dp_bitwise(victim, pi):
    """Fail-stop detection with D=2 pipelines of P=2, one node per process:
    the victim's process goes silent and exits; the survivors (its pipeline
    and the other one, which waits in its all-reduce) detect it, agree on the
    cut and recover; every later step equals the failure-free D=2 run bit
    for bit."""
    cfg = get_config("C0")
    D, P = 2, cfg.stages
    losses, state = single_dp(cfg, D, 3)
    ranks = run_mp(4, config="C0", stages=P, steps=3, pipelines=D, failstop=f"1:{victim}:{pi}",
                   detect=300)
    assert ranks[victim] is None
    live = [r for r in ranks if r is not None]
    for t in range(1, 3):   # step 0's share of a last-stage victim left with it
        parts = [np.float32(r["losses"][t]) for r in live if not np.isnan(r["losses"][t])]
        assert len(parts) == D, (t, parts)
        tot = np.float32(0)
        for x in parts:
            tot = np.float32(tot + x)
        assert tot == np.float32(losses[t]), (t, parts, losses[t])
    for w in state:
        assert np.array_equal(merged(live, D * P, w), state[w]), w


@pytest.mark.parametrize("victim,pi", [(-1, 0), (1, 12), (2, 30)])
def test_multi_process_dp_efeb_bitwise(victim, pi):
    """EFEB with D=2 pipelines of P=2 over 4 processes (eager BRC, replicas
    synced with the all-reduced total): equals the single-process run bit
    for bit, also after a preemption."""
    cfg = get_config("C0")
    D, P = 2, cfg.stages
    losses, state = single_dp(cfg, D, 2, rc="efeb")
    extra = {"victim": victim, "pi": pi} if victim >= 0 else {}
    ranks = run_mp(4, config="C0", stages=P, steps=2, pipelines=D, rc="efeb", **extra)
    for t in range(2):
        parts = [np.float32(r["losses"][t]) for r in ranks if not np.isnan(r["losses"][t])]
        tot = np.float32(0)
        for x in parts:
            tot = np.float32(tot + x)
        assert len(parts) == D and tot == np.float32(losses[t]), (t, parts, losses[t])
    for w in state:
        assert np.array_equal(merged(ranks, D * P, w), state[w]), w
