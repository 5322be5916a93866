"""GPU parity of D > 1 data-parallel pipelines through the C ABI (SURVEY.md
§8(f)-3; PAPER.md P:57, P:385 the all-reduce at the end of an iteration,
P:421 it waits for a failed pipeline).

C0 (P=2, M=4, mb=2) as D=2 pipelines on one device (4 nodes): every step
against the fp64 oracle (tests/parity.py tolerances: bf16 1e-2 / fp32 1e-5)
with each pipeline's local gradient sum, Adam m / v and the update (from the
all-reduced total) checked; every pipeline's copy of a stage bit-identical
to the others' (the all-reduce adds in ascending pipeline order on every
pipeline); a preemption in either pipeline at any point recovers to the
failure-free result bit for bit (the other pipeline's all-reduce waits for
the shadow, which replays the victim's); two failures and LIFO rejoin.
"""
import dataclasses

import numpy as np
import pytest

from oracle import pipeline as opipe, plan as opl
from synth import get_config, make_params, make_tokens
from parity import TOL, check_tensors, check_update

pytestmark = pytest.mark.gpu

LR = 1e-4
D = 2
STATES = ("params", "grads", "adam_m", "adam_v")


def _batch(cfg, t):
    return make_tokens(dataclasses.replace(cfg, microbatches=D * cfg.microbatches), t)


def _gpu(cfg, flat, prec="bf16", rc="eflb"):
    import paper_2204_12013_b200 as bb
    p = bb.Pipeline(cfg.model, cfg.stages, cfg.microbatches, micro_batch=cfg.micro_batch, rc=rc,
                    prec=prec, lr=LR, pipelines=D)
    p.load_params(flat)
    return p


def _flat(p, P, what, d):
    return np.concatenate([p.read_state(d * P + s, what) for s in range(P)])


@pytest.mark.parametrize("prec", ["bf16", "fp32"])
def test_dp_steps_match_oracle(prec):
    cfg = get_config("C0")
    P, M = cfg.stages, cfg.microbatches
    flat = make_params(cfg.model)
    p = _gpu(cfg, flat, prec)
    ref = opipe.Pipeline(cfg, flat, rc=True, lr=LR, D=D)
    host, rep = opl.normal_topology(P, D)
    assert p.schedule_dump() == opl.dump(P, M, True, opl.partition(cfg.model.n_layer, P),
                                         opl.normal_plans(P, M, True, D), host, rep)
    lay = ref.lay
    tol = TOL[prec]
    for t in range(3):
        tok, tgt = _batch(cfg, t)
        p0 = np.concatenate([ref.params(X)["p"] for X in range(P)]).astype(np.float32)
        m0 = np.concatenate([ref.params(X)["m"] for X in range(P)])
        v0 = np.concatenate([ref.params(X)["v"] for X in range(P)])
        if t > 0:   # start from the oracle's state (teacher forcing, as in test_gpu_step)
            from synth import round_to_bf16
            if prec == "bf16":
                for node in ref.nodes.values():
                    for c in node.copies.values():
                        c["p"][:] = round_to_bf16(c["p"].astype(np.float32)).astype(np.float64)
                p0 = np.concatenate([ref.params(X)["p"] for X in range(P)]).astype(np.float32)
            for X in range(P):
                lo, hi = ref.stage_bounds(X)
                for what, val in (("params", p0), ("adam_m", m0), ("adam_v", v0)):
                    p.write_state(X, what, np.asarray(val[lo:hi], np.float32))
        status, st = p.step(tok, tgt)
        assert status == "ok"
        _, ref_loss = ref.step(tok, tgt)
        assert abs(st.loss - ref_loss) <= tol * abs(ref_loss), (st.loss, ref_loss)
        total = np.zeros(lay.total, np.float32)
        for d in range(D):   # each pipeline's local gradient sum
            g = _flat(p, P, "grads", d)
            rg = np.concatenate([ref.params(X, d)["g"] for X in range(P)])
            check_tensors(lay, 0, lay.total, g, rg, prec, f"grad[pipe {d}]")
            total = total + g     # the device adds in the same order (fp32)
        for d in range(D):
            m, v = _flat(p, P, "adam_m", d), _flat(p, P, "adam_v", d)
            rm = np.concatenate([ref.params(X, d)["m"] for X in range(P)])
            rv = np.concatenate([ref.params(X, d)["v"] for X in range(P)])
            check_tensors(lay, 0, lay.total, m, rm, prec, "adam_m")
            check_tensors(lay, 0, lay.total, v, rv, prec, "adam_v", factor=2.0)
            check_update(lay, 0, lay.total, _flat(p, P, "params", d), p0, total, m0, v0,
                         t + 1, (LR, 0.9, 0.999, 1e-8))
    p.close()


def _run(cfg, flat, steps, events=None, rc="eflb"):
    p = _gpu(cfg, flat, rc=rc)
    P = cfg.stages
    out, rec = [], []
    for t in range(steps):
        ev = (events or {}).get(t)
        if ev == "rejoin":
            p.rejoin()
        elif ev is not None:
            p.preempt(*ev)
        status, st = p.step(*_batch(cfg, t))
        loss = st.loss
        if status == "preempted":
            r = p.recover()
            loss = r.loss
            rec.append(p.recovery_dump())
        state = {(d, w): _flat(p, P, w, d) for d in range(D) for w in ("params", "adam_m", "adam_v")}
        out.append((loss, state))
    return p, out, rec


def _same(a, b):
    assert a[0] == b[0], (a[0], b[0])
    for k in b[1]:
        assert np.array_equal(a[1][k], b[1][k]), k


@pytest.mark.parametrize("rc", ["eflb", "lflb", "efeb", "none"])
def test_dp_pipelines_bit_identical(rc):
    cfg = get_config("C0")
    flat = make_params(cfg.model)
    p, out, _ = _run(cfg, flat, 3, rc=rc)
    for loss, st in out:
        for w in ("params", "adam_m", "adam_v"):
            assert np.array_equal(st[(0, w)], st[(1, w)]), w
    if rc != "none":
        for g in range(D * cfg.stages):   # replicas too
            for w in ("params", "adam_m", "adam_v"):
                assert np.array_equal(p.read_state(g, w), p.read_state(g, w, replica=True))
    p.close()


@pytest.mark.parametrize("rc", ["eflb", "efeb", "lflb"])
def test_dp_recovery_bitwise_every_node(rc):
    """Each of the 4 nodes at sampled points of the step (incl. before its
    all-reduce, between its sends and receives, after its commit): the
    interrupted step and a failover step equal the failure-free run bit for
    bit, and the recovery dump is the oracle's."""
    cfg = get_config("C0")
    P, M = cfg.stages, cfg.microbatches
    flat = make_params(cfg.model)
    p, ref, _ = _run(cfg, flat, 2, rc=rc)
    p.close()
    plans = opl.normal_plans(P, M, rc, D)
    for v in range(D * P):
        kinds = [i.kind for i in plans[v]]
        n = len(kinds)
        pts = {0, 5, n // 2, kinds.index(opl.AR_SEND), kinds.index(opl.AR_SEND) + 1,
               kinds.index(opl.AR_SUM), kinds.index(opl.REPLICA_SEND) + 1, n}
        for pi in sorted(pts):
            q, out, rec = _run(cfg, flat, 2, events={0: (v, pi)}, rc=rc)
            assert rec[0] == opl.recovery_dump(P, M, v, pi, rc, D=D), (v, pi)
            if np.isnan(out[0][0]):   # LFLB: a last stage lost after its commit
                assert rc == "lflb" and v % P == P - 1   # point took its loss share
                out[0] = (ref[0][0], out[0][1])
            _same(out[0], ref[0])
            _same(out[1], ref[1])
            q.close()


def test_dp_two_failures_and_rejoin_bitwise():
    """Stage 1 of pipeline 0, then stage 1 of pipeline 1 (both all-reduce
    partners of stage 1 are shadows now), LIFO rejoin of both."""
    cfg = get_config("C0")
    flat = make_params(cfg.model)
    p, ref, _ = _run(cfg, flat, 6)
    p.close()
    q, out, _ = _run(cfg, flat, 6, events={0: (1, 11), 1: (3, 20), 3: "rejoin", 4: "rejoin"})
    for t in range(6):
        _same(out[t], ref[t])
    q.close()
