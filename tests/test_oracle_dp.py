"""Pins for D > 1 data-parallel pipelines in the oracle (
PAPER.md P:57 "data-parallel ... each pipeline", P:385 all-reduce at the end
of an iteration, P:421 the all-reduce waits for a failed pipeline).

* D pipelines of P stages on D*M micro-batches == the brute-force single-device
  step on the whole batch (the loss is the batch mean, so the all-reduced sum
  of the per-pipeline gradients is the full-batch gradient): a dropped
  contribution, a wrong token split or a per-pipeline normalisation fails it;
* every pipeline applies the same total: all D copies of a stage (and their
  replicas) are bit-identical after every step;
* a preemption in one pipeline at any point is recovered by its shadow, which
  replays the victim's all-reduce (the other pipelines resend what the victim
  had consumed): every step equals the failure-free run exactly;
* failures in two pipelines (also of the same stage) are two independent
  recoveries; rejoin restores the normal plans.
"""
import dataclasses
import random

import numpy as np
import pytest

from oracle import model, pipeline, plan as pl
from synth import get_config, make_params, make_tokens


def tiny(P, M, L=None, mb=1, S=8, H=16, nh=2, V=32, causal=True):
    c0 = get_config("C0")
    L = P if L is None else L
    m = dataclasses.replace(c0.model, n_layer=L, d_model=H, n_head=nh, d_ff=4 * H, vocab=V,
                            vocab_sample=V, seq_len=S, causal=causal)
    return dataclasses.replace(c0, name="tiny", model=m, stages=P, microbatches=M, micro_batch=mb)


def batch(cfg, D, t):
    """The step's whole batch: D*M micro-batches (pipeline d takes d*M..)."""
    return make_tokens(dataclasses.replace(cfg, microbatches=D * cfg.microbatches), t)


def state(pp, d=0):
    P = pp.P
    return (np.concatenate([pp.params(X, d)["p"] for X in range(P)]),
            np.concatenate([pp.params(X, d)["m"] for X in range(P)]),
            np.concatenate([pp.params(X, d)["v"] for X in range(P)]))


def run(cfg, D, flat, steps, rc="eflb", events=None):
    pp = pipeline.Pipeline(cfg, flat, rc=rc, D=D)
    out = []
    for t in range(steps):
        ev = (events or {}).get(t)
        if ev == "rejoin":
            pp.rejoin()
        elif ev is not None:
            pp.preempt(*ev)
        status, loss = pp.step(*batch(cfg, D, t))
        if status == "preempted":
            loss, _ = pp.recover()
        out.append((loss, *state(pp)))
    return pp, out


def same(a, b):
    assert a[0] == b[0], (a[0], b[0])
    for x, y in zip(a[1:], b[1:]):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("P,M,D,rc", [(2, 2, 2, "none"), (2, 2, 2, "eflb"), (3, 2, 2, "lflb"),
                                      (2, 1, 3, "eflb"), (3, 3, 2, "eflb"), (3, 2, 2, "efeb"),
                                      (2, 2, 2, "efeb")])
def test_dp_equals_brute_force(P, M, D, rc):
    cfg = tiny(P, M)
    flat = make_params(cfg.model)
    lay = model.Layout(cfg.model)
    p, m, v = flat.astype(np.float64), np.zeros(lay.total), np.zeros(lay.total)
    pp = pipeline.Pipeline(cfg, flat, rc=rc, D=D)
    for t in range(1, 3):
        tok, tgt = batch(cfg, D, t - 1)
        loss, g, p, m, v = model.train_step(lay, p, m, v, t, tok, tgt, 1e-4, 0.9, 0.999, 1e-8)
        status, got = pp.step(tok, tgt)
        assert status == "ok"
        assert abs(got - loss) <= 1e-12 * abs(loss)
        # the per-pipeline local sums add up to the full-batch gradient
        local = sum(np.concatenate([pp.params(X, d)["g"] for X in range(P)]) for d in range(D))
        assert np.abs(local - g).max() <= 1e-12 * np.abs(g).max()
        for d in range(D):
            gp, gm, gv = state(pp, d)
            assert np.abs(gp - p).max() <= 1e-12 * np.abs(p).max()
            assert np.abs(gm - m).max() <= 1e-12 * np.abs(m).max()


@pytest.mark.parametrize("rc", ["eflb", "efeb", "lflb"])
def test_dp_pipelines_and_replicas_identical(rc):
    P, M, D = 3, 2, 3
    cfg = tiny(P, M)
    pp = pipeline.Pipeline(cfg, make_params(cfg.model), rc=rc, D=D)
    for t in range(3):
        pp.step(*batch(cfg, D, t))
        for d in range(1, D):
            for a, b in zip(state(pp, 0), state(pp, d)):
                assert np.array_equal(a, b)
        for g in range(P * D):
            s, rep = g % P, pp.replica_on[g]
            for key in ("p", "m", "v"):
                assert np.array_equal(pp.nodes[g].copies[s][key], pp.nodes[rep].copies[s][key])


def test_dp_plan_structure():
    """Each node all-reduces its stage with the same stage of every other
    pipeline after its last backward and before the replica sync."""
    P, M, D = 3, 4, 2
    plans = pl.normal_plans(P, M, "eflb", D)
    assert sorted(plans) == list(range(P * D))
    for n, seq in plans.items():
        kinds = [i.kind for i in seq]
        last_bwd = max(i for i, k in enumerate(kinds) if k == pl.BWD)
        a = kinds.index(pl.AR_SEND)
        assert last_bwd < a < kinds.index(pl.AR_SUM) < kinds.index(pl.REPLICA_SEND)
        peers = {i.peer for i in seq if i.kind in (pl.AR_SEND, pl.AR_RECV)}
        assert peers == {e * P + n % P for e in range(D)} - {n}
        # every other instruction stays inside the pipeline
        for i in seq:
            if i.peer is not None and i.kind not in (pl.AR_SEND, pl.AR_RECV):
                assert i.peer // P == n // P
    pcs, ch = pl.lockstep(plans)
    assert all(pcs[n] == len(plans[n]) for n in plans) and not any(ch.values())


def test_dp_resend_to_shadow():
    """The other pipelines never wait for the victim's pipeline before their
    own AR_SEND, so at any cut before the victim's commit point (its replica
    sync) their contribution to it is lost with it and sent again to the
    shadow, which replays the whole all-reduce; after the commit point the
    victim's all-reduce was complete and nothing is resent."""
    P, M, D = 2, 2, 2
    plans = pl.normal_plans(P, M, "eflb", D)
    v = 1
    seq = plans[v]
    after_recv = max(i for i, x in enumerate(seq) if x.kind == pl.AR_RECV) + 1
    commit = [x.kind for x in seq].index(pl.REPLICA_SEND) + 1
    for pi, resend in ((0, True), (after_recv, True), (commit, False)):
        pcs, ch = pl.cut(plans, v, pi)
        new, info = pl.recovery_plans(plans, P, M, v, pcs, ch)
        o = P + v % P                         # pipeline 1's node of the victim's stage
        got = [i for i in new[o] if i.kind == pl.RESEND_AR]
        assert bool(got) == resend and all(i.peer == info["shadow"] for i in got)
        assert all(i.peer != v for i in new[o])
        p2, c2 = pl.lockstep(new, {n: 0 for n in new}, ch)
        assert all(p2[n] == len(new[n]) for n in new)
        assert not any(c2.values())             # no message left unconsumed


def test_dp_injection_sweep_exact():
    """Every node of a D=2 x P=2 (and a sample of D=2 x P=3) run, injection
    points sampled over the whole step: the interrupted step and the next one
    (failover plans) equal the failure-free run exactly."""
    r = random.Random(7)
    for P, M, D, per in ((2, 2, 2, None), (3, 2, 2, 6)):
        cfg = tiny(P, M)
        flat = make_params(cfg.model)
        _, ref = run(cfg, D, flat, 2)
        plans = pl.normal_plans(P, M, "eflb", D)
        for v in range(P * D):
            n = len(plans[v])
            pts = range(n + 1) if per is None else sorted({0, n} | {r.randint(0, n) for _ in range(per)})
            for pi in pts:
                pp, res = run(cfg, D, flat, 2, events={0: (v, pi)})
                same(res[0], ref[0])
                same(res[1], ref[1])
                assert pp.mode == "failover"
                for d in range(D):   # every pipeline applied the same update
                    for a, b in zip(state(pp, 0), state(pp, d)):
                        assert np.array_equal(a, b)


def test_dp_two_pipelines_fail_and_rejoin_exact():
    """Lose stage 1 of pipeline 0, then stage 1 of pipeline 1 (the same stage:
    its all-reduce partner is now a shadow), then rejoin both (LIFO)."""
    P, M, D = 3, 2, 2
    cfg = tiny(P, M)
    flat = make_params(cfg.model)
    _, ref = run(cfg, D, flat, 6)
    plans = pl.normal_plans(P, M, "eflb", D)
    r = random.Random(1)
    for v2 in (P + 1, P + 0, P + 2):
        ev = {0: (1, r.randint(0, len(plans[1]))), 3: "rejoin", 4: "rejoin"}
        pp = pipeline.Pipeline(cfg, flat, rc="eflb", D=D)
        for t in range(6):
            e = ev.get(t)
            if e == "rejoin":
                pp.rejoin()
            elif e is not None:
                pp.preempt(*e)
            if t == 1:
                pp.preempt(v2, r.randint(0, len(pp.plans[v2])))
            status, loss = pp.step(*batch(cfg, D, t))
            if status == "preempted":
                loss, info = pp.recover()
            same((loss, *state(pp)), ref[t])
            same((loss, *state(pp, 1)), ref[t])
        assert pp.mode == "normal" and not pp.victims


def test_dp_recovery_dump_golden_shape():
    """The recovery dump of a D>1 cut names the pipeline-local shadow."""
    txt = pl.recovery_dump(2, 2, 3, 5, "eflb", D=2)
    assert txt.startswith("# bamboo-recovery v1 P=2 M=2 victim=3 shadow=2 successor=2")


@pytest.mark.parametrize("mode", ["efeb", "lflb"])
def test_dp_modes_injection_sweep_exact(mode):
    """EFEB and LFLB with D = 2: every node, sampled points; exact equality
    with the failure-free run on the interrupted and the next step."""
    r = random.Random(17)
    for P, M in ((2, 2), (3, 2)):
        cfg = tiny(P, M)
        flat = make_params(cfg.model)
        _, ref = run(cfg, 2, flat, 2, rc=mode)
        plans = pl.normal_plans(P, M, mode, 2)
        for v in range(2 * P):
            n = len(plans[v])
            for pi in sorted({0, n, n // 2} | {r.randint(0, n) for _ in range(4)}):
                _, res = run(cfg, 2, flat, 2, rc=mode, events={0: (v, pi)})
                if np.isnan(res[0][0]):   # LFLB: a last stage lost after its commit point
                    assert mode == "lflb" and v % P == P - 1   # took its losses with it
                    res[0] = (ref[0][0],) + tuple(res[0][1:])
                same(res[0], ref[0])
                same(res[1], ref[1])
