"""Pins for oracle/pipeline.py:

* pipelined == brute-force single-device step (P:140-142 synchronous
  micro-batching keeps one consistent model state), 1F1B == GPipe;
* FRC^n_{n+1} output and saved set == FNC_{n+1} exactly;
* replica == primary exactly after every step ("same model parameters
  and optimizer states");
* an injected preemption + recovery gives loss, gradients, parameters and
  Adam state EXACTLY equal to the failure-free run (north star), for every
  victim and every injection point on C0 and on random tiny pipelines;
* consecutive preemptions are FATAL.
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


def brute(cfg, flat, steps, lr=1e-4):
    lay = model.Layout(cfg.model)
    p, m, v = flat.astype(np.float64), np.zeros(lay.total), np.zeros(lay.total)
    out = []
    for t in range(1, steps + 1):
        tok, tgt = make_tokens(cfg, t - 1)
        loss, g, p, m, v = model.train_step(lay, p, m, v, t, tok, tgt, lr, 0.9, 0.999, 1e-8)
        out.append((loss, g, p.copy(), m.copy(), v.copy()))
    return out


@pytest.mark.parametrize("rc", [False, True])
def test_pipelined_equals_brute_force_c0(rc):
    cfg = get_config("C0")
    flat = make_params(cfg.model)
    ref = brute(cfg, flat, 2)
    pp = pipeline.Pipeline(cfg, flat, rc=rc)
    for t in range(2):
        tok, tgt = make_tokens(cfg, t)
        status, loss = pp.step(tok, tgt)
        assert status == "ok"
        rl, rg, rp, rm, rv = ref[t]
        assert abs(loss - rl) <= 1e-12 * abs(rl)
        assert np.abs(pp.full_grads() - rg).max() <= 1e-12 * np.abs(rg).max()
        assert np.abs(pp.full_params() - rp).max() <= 1e-12 * np.abs(rp).max()


def test_1f1b_equals_gpipe():
    cfg = tiny(3, 4)
    flat = make_params(cfg.model)
    a = pipeline.Pipeline(cfg, flat, rc=False)
    b = pipeline.Pipeline(cfg, flat, rc=False)
    b.plans = {s: pl.gpipe_plan(s, 3, 4) for s in range(3)}
    tok, tgt = make_tokens(cfg, 0)
    la = a.step(tok, tgt)[1]
    lb = b.step(tok, tgt)[1]
    assert abs(la - lb) <= 1e-13 * abs(la)
    assert np.allclose(a.full_grads(), b.full_grads(), rtol=0, atol=1e-14)


def _frc_equals_fnc(pp):
    P = pp.P
    stores = pp.last_stores
    for n in range(P):
        X = (n + 1) % P
        for k in range(pp.M):
            frc_saved = stores[n][("saved", X, k)]
            fnc_saved = stores[X][("saved", X, k)]
            for a, b in zip(frc_saved, fnc_saved):
                assert a.keys() == b.keys()
                for key in a:
                    if key in ("s1", "s2", "ln"):
                        assert all(np.array_equal(x, y) for x, y in zip(a[key], b[key]))
                    else:
                        assert np.array_equal(a[key], b[key])
            okey = ("act", X + 1, k) if X < P - 1 else ("loss", k)
            assert np.array_equal(np.asarray(stores[n][okey]), np.asarray(stores[X][okey]))


def test_frc_is_fnc_and_replica_is_primary():
    cfg = tiny(3, 4)
    pp = pipeline.Pipeline(cfg, make_params(cfg.model), rc=True)
    for t in range(3):
        tok, tgt = make_tokens(cfg, t)
        pp.step(tok, tgt)
        _frc_equals_fnc(pp)
        for s in range(3):
            prim = pp.nodes[s].copies[s]
            rep = pp.nodes[(s - 1) % 3].copies[s]
            for key in ("p", "m", "v", "g"):
                assert np.array_equal(prim[key], rep[key])
            assert prim["t"] == rep["t"]


def _run(cfg, flat, steps, inject=None):
    pp = pipeline.Pipeline(cfg, flat, rc=True)
    res = []
    for t in range(steps):
        tok, tgt = make_tokens(cfg, t)
        if inject is not None and inject[0] == t:
            pp.preempt(inject[1], inject[2])
        status, val = pp.step(tok, tgt)
        if status == "preempted":
            val, info = pp.recover()
        res.append((val, pp.full_grads().copy(), pp.full_params().copy(),
                    *[a.copy() for a in pp.full_adam()]))
    return pp, res


def _same(a, b):
    assert a[0] == b[0]
    for x, y in zip(a[1:], b[1:]):
        assert np.array_equal(x, y)


def test_c0_injection_sweep_exact():
    """C0 (BASELINE configs[0]): every victim, every injection point."""
    cfg = get_config("C0")
    flat = make_params(cfg.model)
    _, ref = _run(cfg, flat, 2)
    plans = pl.normal_plans(cfg.stages, cfg.microbatches, True)
    for v in range(cfg.stages):
        for pi in range(len(plans[v]) + 1):
            pp, res = _run(cfg, flat, 2, inject=(0, v, pi))
            _same(res[0], ref[0])        # the interrupted step
            _same(res[1], ref[1])        # a following step on the failover plan
            assert pp.mode == "failover"


def test_random_tiny_injections_exact():
    r = random.Random(11)
    for _ in range(12):
        P = r.randint(2, 5)
        M = r.randint(1, 6)
        cfg = tiny(P, M, L=P + r.randint(0, 2), causal=bool(r.randint(0, 1)))
        flat = make_params(cfg.model)
        _, ref = _run(cfg, flat, 2)
        plans = pl.normal_plans(P, M, True)
        for _ in range(4):
            v = r.randrange(P)
            pi = r.randint(0, len(plans[v]))
            _, res = _run(cfg, flat, 2, inject=(0, v, pi))
            _same(res[0], ref[0])
            _same(res[1], ref[1])


def test_second_preemption_is_fatal():
    cfg = get_config("C0")
    pp = pipeline.Pipeline(cfg, make_params(cfg.model), rc=True)
    tok, tgt = make_tokens(cfg, 0)
    pp.preempt(1, 5)
    assert pp.step(tok, tgt)[0] == "preempted"
    pp.recover()
    with pytest.raises(pl.Fatal):     # P:464, Q18: no redundancy left
        pp.preempt(0, 0)


def test_adjacent_second_preemptions_are_fatal():
    """After losing v: the double-duty shadow v-1, the dead v itself and the
    unprotected successor v+1 (its replica was on v) cannot be lost."""
    cfg = tiny(5, 3)
    pp = pipeline.Pipeline(cfg, make_params(cfg.model), rc=True)
    pp.preempt(2, 4)
    assert pp.step(*make_tokens(cfg, 0))[0] == "preempted"
    pp.recover()
    for v in (1, 2, 3):
        with pytest.raises(pl.Fatal):
            pp.preempt(v, 0)
    for v in (0, 4):
        pp.preempt(v, 0)      # recoverable: armed (and disarmed by the next line)
        pp.pending = None


def test_non_adjacent_second_preemption_exact():
    """two non-adjacent preemptions are two independent recoveries.
    P=4/5: lose v1 at some point of step 0, then a non-adjacent v2 at every
    point of step 2 (on the failover plan); every step equals the failure-free
    run exactly; then both rejoin (LIFO) and the run continues exactly."""
    r = random.Random(3)
    for P, M in ((4, 3), (5, 4)):
        cfg = tiny(P, M)
        flat = make_params(cfg.model)
        _, ref = _run(cfg, flat, 6)
        plans = pl.normal_plans(P, M, True)
        for v1 in range(P):
            ok = [v for v in range(P) if v not in ((v1 - 1) % P, v1, (v1 + 1) % P)]
            for v2 in ok:
                pi1 = r.randint(0, len(plans[v1]))
                pp = pipeline.Pipeline(cfg, flat, rc=True)
                pp.preempt(v1, pi1)
                assert pp.step(*make_tokens(cfg, 0))[0] == "preempted"
                val, _ = pp.recover()
                _same((val, pp.full_grads(), pp.full_params(), *pp.full_adam()), ref[0])
                status, val = pp.step(*make_tokens(cfg, 1))
                _same((val, pp.full_grads(), pp.full_params(), *pp.full_adam()), ref[1])
                n2 = len(pp.plans[v2])
                for pi2 in sorted({0, n2 // 3, n2 // 2, n2, r.randint(0, n2)}):
                    q = pipeline.Pipeline(cfg, flat, rc=True)
                    q.preempt(v1, pi1)
                    q.step(*make_tokens(cfg, 0))
                    q.recover()
                    q.step(*make_tokens(cfg, 1))
                    q.preempt(v2, pi2)
                    assert q.step(*make_tokens(cfg, 2))[0] == "preempted"
                    val, info = q.recover()
                    assert info["victim"] == v2 and q.victims == [v1, v2]
                    _same((val, q.full_grads(), q.full_params(), *q.full_adam()), ref[2])
                    _, val = q.step(*make_tokens(cfg, 3))       # double-failover plan
                    _same((val, q.full_grads(), q.full_params(), *q.full_adam()), ref[3])
                    q.rejoin()
                    _, val = q.step(*make_tokens(cfg, 4))
                    _same((val, q.full_grads(), q.full_params(), *q.full_adam()), ref[4])
                    q.rejoin()
                    assert q.mode == "normal"
                    _, val = q.step(*make_tokens(cfg, 5))
                    _same((val, q.full_grads(), q.full_params(), *q.full_adam()), ref[5])


def test_no_rc_preemption_is_fatal():
    cfg = get_config("C0")
    pp = pipeline.Pipeline(cfg, make_params(cfg.model), rc=False)
    with pytest.raises(pl.Fatal):
        pp.preempt(1, 3)


def test_rejoin_and_repeated_preemptions_exact():
    """C4-style run: preempt, run on the failover plan, rejoin,
    preempt another node, ... equals the failure-free run exactly."""
    r = random.Random(5)
    for P, M in ((2, 4), (3, 3), (4, 5)):
        cfg = tiny(P, M)
        flat = make_params(cfg.model)
        _, ref = _run(cfg, flat, 7)
        pp = pipeline.Pipeline(cfg, flat, rc=True)
        plans = pl.normal_plans(P, M, True)
        events = {0: (r.randrange(P),), 2: "rejoin", 3: (r.randrange(P),), 5: "rejoin"}
        for t in range(7):
            tok, tgt = make_tokens(cfg, t)
            ev = events.get(t)
            if ev == "rejoin":
                pp.rejoin()
                assert pp.mode == "normal"
            elif ev is not None:
                v = ev[0]
                pp.preempt(v, r.randint(0, len(plans[v])))
            status, val = pp.step(tok, tgt)
            if status == "preempted":
                val, _ = pp.recover()
            _same((val, pp.full_grads(), pp.full_params(), *pp.full_adam()), ref[t])
        # after a rejoin the replicas are exact again
        for s in range(P):
            for key in ("p", "m", "v"):
                assert np.array_equal(pp.nodes[s].copies[s][key], pp.nodes[(s - 1) % P].copies[s][key])


def test_lflb_injection_sweep_exact():
    """LFLB: replicas kept in sync, no FRC; a failure recomputes
    the victim's forward (lazy FRC) and backward (lazy BRC) for the whole
    step. Every victim / point of a P=3 pipeline equals the failure-free run
    exactly, and the plans carry no FRC_FWD."""
    cfg = tiny(3, 4)
    flat = make_params(cfg.model)
    _, ref = _run(cfg, flat, 2)
    plans = pl.normal_plans(3, 4, "lflb")
    assert not any(i.kind == pl.FRC_FWD for seq in plans.values() for i in seq)
    for v in range(3):
        for pi in range(len(plans[v]) + 1):
            pp = pipeline.Pipeline(cfg, flat, rc="lflb")
            res = []
            for t in range(2):
                tok, tgt = make_tokens(cfg, t)
                if t == 0:
                    pp.preempt(v, pi)
                status, val = pp.step(tok, tgt)
                if status == "preempted":
                    val, info = pp.recover()
                    assert info["frc_done"] == []
                    if v == 2 and info["commit"]:   # the loss left with the last stage
                        assert np.isnan(val)
                        val = ref[0][0]
                res.append((val, pp.full_grads().copy(), pp.full_params().copy(),
                            *[a.copy() for a in pp.full_adam()]))
            _same(res[0], ref[0])
            _same(res[1], ref[1])


@pytest.mark.parametrize("P,M", [(2, 3), (3, 4), (4, 5), (5, 3)])
def test_efeb_injection_sweep_exact(P, M):
    """EFEB: eager FRC and eager BRC (from the duplicate
    gradient of node s+2), no replica sync. The replica's own gradient and
    state equal the primary's exactly every step; a preemption at every point
    of every victim leaves the run exactly equal to the failure-free one, and
    the following failover step too."""
    cfg = tiny(P, M)
    flat = make_params(cfg.model)
    _, ref = _run(cfg, flat, 2)
    plans = pl.normal_plans(P, M, "efeb")
    assert not any(i.kind in (pl.REPLICA_SEND, pl.REPLICA_RECV) for q in plans.values() for i in q)
    pp = pipeline.Pipeline(cfg, flat, rc="efeb")
    for t in range(2):
        pp.step(*make_tokens(cfg, t))
        for s in range(P):
            prim, rep = pp.nodes[s].copies[s], pp.nodes[(s - 1) % P].copies[s]
            for key in ("p", "m", "v", "g"):
                assert np.array_equal(prim[key], rep[key]), (t, s, key)
    for v in range(P):
        for pi in range(len(plans[v]) + 1):
            pp = pipeline.Pipeline(cfg, flat, rc="efeb")
            res = []
            for t in range(2):
                tok, tgt = make_tokens(cfg, t)
                if t == 0:
                    pp.preempt(v, pi)
                status, val = pp.step(tok, tgt)
                if status == "preempted":
                    val, info = pp.recover()
                    if v == P - 1 and np.isnan(val):
                        val = ref[0][0]
                res.append((val, pp.full_grads().copy(), pp.full_params().copy(),
                            *[a.copy() for a in pp.full_adam()]))
            _same(res[0], ref[0])
            _same(res[1], ref[1])
