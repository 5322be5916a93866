"""GPU parity of the full hot path through the C ABI (run under gpurun).

C0 = BASELINE configs[0] (4 layers, H=64, 2 heads, S=32, P=2, M=4, mb=2) runs
with both stages on cuda:0 (stages > GPUs share one device). Checked against
the fp64 oracle on the same seeded inputs (tests/parity.py, north star
"max relative error 1e-2 (bf16) / 1e-5 (fp32)"): plan dump byte-equal; loss,
every gradient tensor, Adam m and v and the parameter update of EVERY step
(each step starts from the oracle's state: bb_write_state); FRC replica ==
primary bit for bit; preempted + recovered == failure-free bit for bit (the
victim's memory is NaN-poisoned at the injection) and within tolerance of the
oracle. PT1 / PT2: full C1 depth and C2 / C3 width against
oracle fixtures (tools/make_oracle_fixtures.py), failure-free and injected.
"""
import dataclasses
import os

import numpy as np
import pytest

from oracle import pipeline as opipe, plan as opl
from synth import get_config, make_params, make_tokens
from parity import TOL, check_tensors, check_update, check_sampled, tol_for

pytestmark = pytest.mark.gpu

LR = 1e-4
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
STATES = ("params", "grads", "adam_m", "adam_v")


def _gpu(cfg, flat, prec, rc=True, **kw):
    import paper_2204_12013_b200 as bb
    p = bb.Pipeline(cfg.model, cfg.stages, cfg.microbatches, micro_batch=cfg.micro_batch, rc=rc,
                    prec=prec, lr=LR, **kw)
    p.load_params(flat)
    return p


def _flat_state(p, P, what):
    return np.concatenate([p.read_state(s, what) for s in range(P)])


def _force_oracle_state(p, ref, P, prec):
    """Start the next GPU step from the oracle's state (params, m, v). In bf16
    the oracle's parameters are first rounded to bf16-representable values on
    the oracle side too (every copy), so both sides start from identical
    numbers (Q16) and the GPU's bf16 working copy adds no rounding."""
    from synth import round_to_bf16
    if prec == "bf16":
        for node in ref.nodes.values():
            for c in node.copies.values():
                c["p"][:] = round_to_bf16(c["p"].astype(np.float32)).astype(np.float64)
    m, v = ref.full_adam()
    for X in range(P):
        lo, hi = ref.stage_bounds(X)
        for what, val in (("params", ref.full_params()), ("adam_m", m), ("adam_v", v)):
            p.write_state(X, what, val[lo:hi])


def _state0(ref):
    """The oracle's (params, m, v, Adam step) before a step."""
    m, v = ref.full_adam()
    return ref.full_params().copy(), m.copy(), v.copy(), ref.step_no


def _compare_step(cfg, p, ref, prec, loss, ref_loss, s0):
    """One step, both sides started from the same state s0 = (p, m, v, t)."""
    tol = TOL[prec]
    lay = ref.lay
    p0, m0, v0, t0 = s0
    assert abs(loss - ref_loss) <= tol * abs(ref_loss), (loss, ref_loss)
    g = _flat_state(p, cfg.stages, "grads")
    rg = ref.full_grads()
    errs = check_tensors(lay, 0, lay.total, g, rg, prec, "grad")
    m, v = _flat_state(p, cfg.stages, "adam_m"), _flat_state(p, cfg.stages, "adam_v")
    rm, rv = ref.full_adam()
    check_tensors(lay, 0, lay.total, m, rm, prec, "adam_m")
    check_tensors(lay, 0, lay.total, v, rv, prec, "adam_v", factor=2.0)
    check_update(lay, 0, lay.total, _flat_state(p, cfg.stages, "params"), p0, g, m0, v0,
                 t0 + 1, (LR, 0.9, 0.999, 1e-8))
    return errs


@pytest.mark.parametrize("prec", ["bf16", "fp32"])
@pytest.mark.parametrize("rc", [True, False])
def test_c0_steps_match_oracle(prec, rc):
    cfg = get_config("C0")
    flat = make_params(cfg.model)
    p = _gpu(cfg, flat, prec, rc)
    ref = opipe.Pipeline(cfg, flat, rc=rc, lr=LR)
    want = opl.dump(cfg.stages, cfg.microbatches, rc, opl.partition(cfg.model.n_layer, cfg.stages),
                    opl.normal_plans(cfg.stages, cfg.microbatches, rc))
    assert p.schedule_dump() == want
    for t in range(3):
        tok, tgt = make_tokens(cfg, t)
        s0 = _state0(ref)
        status, st = p.step(tok, tgt)
        assert status == "ok"
        _, ref_loss = ref.step(tok, tgt)
        _compare_step(cfg, p, ref, prec, st.loss, ref_loss, s0)
        assert st.gpu_launches > 0
        if rc:   # replica == primary, bit for bit
            for s in range(cfg.stages):
                for what in STATES:
                    assert np.array_equal(p.read_state(s, what),
                                          p.read_state(s, what, replica=True)), (t, s, what)
        _force_oracle_state(p, ref, cfg.stages, prec)
    p.close()


@pytest.mark.parametrize("prec", ["bf16", "fp32"])
def test_c0_trajectory_loss(prec):
    """Free-running (no state forcing) for 4 steps: the losses stay within
    the tolerance of the oracle's trajectory."""
    cfg = get_config("C0")
    flat = make_params(cfg.model)
    p = _gpu(cfg, flat, prec)
    ref = opipe.Pipeline(cfg, flat, rc=True, lr=LR)
    for t in range(4):
        tok, tgt = make_tokens(cfg, t)
        _, st = p.step(tok, tgt)
        _, rl = ref.step(tok, tgt)
        assert abs(st.loss - rl) <= TOL[prec] * abs(rl), (t, st.loss, rl)
    p.close()


@pytest.mark.parametrize("prec", ["bf16", "fp32"])
def test_bidirectional_and_three_stages(prec):
    c0 = get_config("C0")
    cfg = dataclasses.replace(c0, model=dataclasses.replace(c0.model, causal=False, n_layer=5),
                              stages=3, microbatches=5, gpt=False)
    flat = make_params(cfg.model)
    p = _gpu(cfg, flat, prec)
    ref = opipe.Pipeline(cfg, flat, rc=True, lr=LR)
    tok, tgt = make_tokens(cfg, 0)
    s0 = _state0(ref)
    _, st = p.step(tok, tgt)
    _, ref_loss = ref.step(tok, tgt)
    _compare_step(cfg, p, ref, prec, st.loss, ref_loss, s0)
    p.close()


def _run(cfg, flat, prec, steps, inject=None, **kw):
    p = _gpu(cfg, flat, prec, **kw)
    out = []
    rec = None
    for t in range(steps):
        tok, tgt = make_tokens(cfg, t)
        if inject is not None and inject[0] == t:
            p.preempt(inject[1], inject[2])
        status, st = p.step(tok, tgt)
        loss = st.loss
        if status == "preempted":
            rec = p.recover()
            loss = rec.loss
        out.append((loss, {w: _flat_state(p, cfg.stages, w) for w in STATES}))
    return p, out, rec


@pytest.mark.parametrize("prec", ["bf16"])
def test_c0_preemption_recovery_bitwise(prec):
    """BASELINE configs[0]: 'one injected preemption of stage 1' — and every
    other (victim, point) of C0: the recovered run equals the failure-free run
    bit for bit (the victim's memory is NaN at the injection, so nothing in the
    recovery reads it), and the continuation plan equals the oracle's."""
    cfg = get_config("C0")
    flat = make_params(cfg.model)
    _, ref, _ = _run(cfg, flat, prec, 2)
    plans = opl.normal_plans(cfg.stages, cfg.microbatches, True)
    for v in range(cfg.stages):
        for pi in range(0, len(plans[v]) + 1):
            p, got, rec = _run(cfg, flat, prec, 2, inject=(0, v, pi))
            assert rec.victim == v and rec.shadow == (v - 1) % cfg.stages
            assert p.recovery_dump() == opl.recovery_dump(cfg.stages, cfg.microbatches, v, pi)
            for (la, sa), (lb, sb) in zip(got, ref):
                assert la == lb, (v, pi)
                for w in sa:
                    assert np.array_equal(sa[w], sb[w]), (v, pi, w)
            host, rep = opl.failover_topology(cfg.stages, v)
            want = opl.dump(cfg.stages, cfg.microbatches, True, opl.partition(4, 2),
                            opl.failover_plans(cfg.stages, cfg.microbatches, v), host, rep,
                            mode="failover", victim=v)
            assert p.schedule_dump() == want
            p.close()


def test_recovered_run_matches_oracle():
    """fp32: the interrupted + recovered step, then a failover step, each
    against the oracle (started from the oracle's state) at 1e-5."""
    cfg = get_config("C0")
    flat = make_params(cfg.model)
    p = _gpu(cfg, flat, "fp32")
    ref = opipe.Pipeline(cfg, flat, rc=True, lr=LR)
    for t in range(2):
        tok, tgt = make_tokens(cfg, t)
        s0 = _state0(ref)
        if t == 0:
            p.preempt(1, 9)
            assert p.step(tok, tgt)[0] == "preempted"
            loss = p.recover().loss
            ref.preempt(1, 9)
            ref.step(tok, tgt)
            rl, _ = ref.recover()
        else:
            _, st = p.step(tok, tgt)
            loss = st.loss
            _, rl = ref.step(tok, tgt)
        _compare_step(cfg, p, ref, "fp32", loss, rl, s0)
        _force_oracle_state(p, ref, cfg.stages, "fp32")
    p.close()


def test_fatal_second_preemption():
    import paper_2204_12013_b200 as bb
    cfg = get_config("C0")
    p, _, _ = _run(cfg, make_params(cfg.model), "bf16", 1, inject=(0, 1, 3))
    with pytest.raises(bb.BambooError) as e:
        p.preempt(0, 0)
    assert e.value.status == bb.BB_E_FATAL   # the shadow holds both stages
    p.close()


def _fixture(name):
    path = os.path.join(GOLDEN, f"{name}.npz")
    if not os.path.exists(path):
        pytest.fail(f"{path} missing: run tools/make_oracle_fixtures.py {name}")
    return dict(np.load(path))


def _fixture_cfg(name):
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "_mof", os.path.join(os.path.dirname(GOLDEN), "..", "tools", "make_oracle_fixtures.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.cases()[name]


def _check_fixture(fix, lay, cfg, p, loss, prec="bf16"):
    assert abs(loss - float(fix["loss"])) <= TOL[prec] * abs(float(fix["loss"])), loss
    st = {w: _flat_state(p, cfg.stages, w) for w in STATES}
    worst = {}
    for _, name, shape, off in lay.entries:
        idx = fix[f"{name}|idx"] + off
        worst[name] = check_sampled(fix, name, "g", st["grads"][idx], prec)
        check_sampled(fix, name, "m", st["adam_m"][idx], prec)
        check_sampled(fix, name, "v", st["adam_v"][idx], prec, factor=2.0)
        # the update: the oracle's Adam (step 1, zero state) on the GPU's own
        # gradient at the sampled elements (parity.check_update)
        from oracle.model import adam_update
        p0 = fix[f"{name}|p0"]
        pe, _, _ = adam_update(p0, st["grads"][idx].astype(np.float64), np.zeros_like(p0),
                               np.zeros_like(p0), 1, LR, 0.9, 0.999, 1e-8)
        bound = 2 * np.spacing(np.abs(pe).astype(np.float32)) + 1e-5 * np.abs(pe - p0)
        assert np.all(np.abs(st["params"][idx] - pe) <= bound), name
    return worst


@pytest.mark.parametrize("name", ["pt1_c1", "pt2_c2", "pt2_c3"])
def test_pt_full_width_matches_oracle(name):
    """PT1 (all 12 C1 layers on 4 stages, 8 micro-batches of 1) and PT2 (C2:
    bidirectional, S=512, H=1024, V=30528; C3: H=1600, 25 heads, FFN 6400,
    S=1024, V=50304; one block per stage, 8 stages): one failure-free step and
    one step with the victim P/2 preempted at its ceil(M/2)-th BWD, both
    against the oracle fixture; the injected step also bit-equal to the
    failure-free one."""
    from oracle import model as om
    fix = _fixture(name)
    cfg = _fixture_cfg(name)
    lay = om.Layout(cfg.model)
    flat = make_params(cfg.model)
    p, got, _ = _run(cfg, flat, "bf16", 1)
    _check_fixture(fix, lay, cfg, p, got[0][0])
    p.close()
    v = cfg.stages // 2
    plan = opl.normal_plans(cfg.stages, cfg.microbatches, True)[v]
    bwds = [i for i, ins in enumerate(plan) if ins.kind == opl.BWD]
    pi = bwds[-(-cfg.microbatches // 2) - 1]
    q, got2, rec = _run(cfg, flat, "bf16", 1, inject=(0, v, pi))
    assert rec.victim == v and rec.brc_mb > 0
    assert got2[0][0] == got[0][0]
    for w in STATES:
        assert np.array_equal(got2[0][1][w], got[0][1][w]), w
    q.close()


def test_c0_rejoin_and_repeated_preemptions_bitwise():
    """C4-style sequence on the GPU: preempt, failover steps, rejoin,
    preempt another node, rejoin... == failure-free run, bit for bit; the
    dumps after a rejoin are the normal plans again."""
    cfg = get_config("C0")
    flat = make_params(cfg.model)
    _, ref, _ = _run(cfg, flat, "bf16", 6)
    p = _gpu(cfg, flat, "bf16")
    events = {0: (1, 9), 2: "rejoin", 3: (0, 17), 5: "rejoin"}
    for t in range(6):
        tok, tgt = make_tokens(cfg, t)
        ev = events.get(t)
        if ev == "rejoin":
            p.rejoin()
        elif ev is not None:
            p.preempt(*ev)
        status, st = p.step(tok, tgt)
        loss = p.recover().loss if status == "preempted" else st.loss
        assert loss == ref[t][0], t
        for w in STATES:
            assert np.array_equal(_flat_state(p, cfg.stages, w), ref[t][1][w]), (t, w)
    want = opl.dump(cfg.stages, cfg.microbatches, True, opl.partition(4, 2),
                    opl.normal_plans(cfg.stages, cfg.microbatches, True))
    assert p.schedule_dump() == want
    for s in range(cfg.stages):   # protection restored: replica == primary again
        assert np.array_equal(p.read_state(s, "params"), p.read_state(s, "params", replica=True))
    p.close()


def test_rejoin_after_reload_keeps_replica_identical():
    """bb_load_params resets every copy's Adam step; a preempt / recover /
    rejoin after a reload must give the returning copies the same step count
    as the copies that stayed (replica == primary afterwards, bit for bit)."""
    cfg = dataclasses.replace(get_config("C0"), stages=3, microbatches=4)
    flat = make_params(cfg.model)
    p = _gpu(cfg, flat, "bf16")
    for t in range(3):
        p.step(*make_tokens(cfg, t))
    p.load_params(flat)
    p.step(*make_tokens(cfg, 3))
    p.preempt(1, 5)
    assert p.step(*make_tokens(cfg, 4))[0] == "preempted"
    p.recover()
    p.rejoin()
    for t in (5, 6):
        p.step(*make_tokens(cfg, t))
    for s in range(cfg.stages):
        for w in STATES:
            assert np.array_equal(p.read_state(s, w), p.read_state(s, w, replica=True)), (s, w)
    p.close()


def test_token_ids_out_of_range_rejected():
    import paper_2204_12013_b200 as bb
    cfg = get_config("C0")
    p = _gpu(cfg, make_params(cfg.model), "bf16")
    tok, tgt = make_tokens(cfg, 0)
    for bad_tok, bad_tgt in ((tok.copy(), tgt), (tok, tgt.copy())):
        (bad_tok if bad_tok is not tok else bad_tgt)[1, 3] = cfg.model.vocab
        with pytest.raises(bb.BambooError) as e:
            p.step(bad_tok, bad_tgt)
        assert e.value.status == bb.BB_E_INVAL
    with pytest.raises(bb.BambooError):
        bad = tok.copy()
        bad[0, 0] = -1
        p.stage_inputs(bad, tgt)
    assert p.step(tok, tgt)[0] == "ok"   # the context is still usable
    p.close()


@pytest.mark.parametrize("budget", [1, "one", "two"])
def test_frc_retention_budget_recovery_bitwise(budget):
    """frc_retain_bytes (Q10): FRC saved sets beyond the budget keep
    only the stage input; the lazy BRC recomputes their forward. Results are
    bit-identical to full retention for every victim and several points, and
    the recovery reports the re-forwards."""
    cfg = dataclasses.replace(get_config("C0"), stages=3, microbatches=6)
    flat = make_params(cfg.model)
    _, ref, _ = _run(cfg, flat, "bf16", 2)
    if budget != 1:   # one / two saved sets of the largest stage
        probe = _gpu(cfg, flat, "bf16")
        slot = max(probe.stage_memory(s)[0] for s in range(cfg.stages))
        probe.close()
        budget = slot * (1 if budget == "one" else 2)
    probe = _gpu(cfg, flat, "bf16", frc_retain_bytes=budget)
    mem = [probe.stage_memory(s) for s in range(cfg.stages)]
    probe.close()
    assert [k for _, k in mem] == [min(cfg.microbatches, budget // b) for b, _ in mem], mem
    plans = opl.normal_plans(cfg.stages, cfg.microbatches, True)
    for v in range(cfg.stages):
        for pi in (3, len(plans[v]) // 2, len(plans[v]) - 6):
            p, got, rec = _run(cfg, flat, "bf16", 2, inject=(0, v, pi), frc_retain_bytes=budget)
            for (la, sa), (lb, sb) in zip(got, ref):
                assert la == lb, (v, pi)
                for w in sa:
                    assert np.array_equal(sa[w], sb[w]), (v, pi, w)
            if budget == 1 and rec.brc_mb > 0:
                assert rec.frc_recomputed_mb >= rec.brc_mb - rec.frc_done_mb, (v, pi)
            p.close()


@pytest.mark.parametrize("host_sets", [2, 100])
def test_frc_host_swap_recovery_bitwise(host_sets):
    """Host-swap tier (frc_swap_bytes, "swap out these data"): with one
    saved set in HBM, the next `host_sets` FRC saved sets go to pinned host
    memory and a lazy BRC copies them back; the rest (if any) are recomputed.
    Bit-identical to full retention for every victim; the recovery reports
    the saved sets it brought back."""
    cfg = dataclasses.replace(get_config("C0"), stages=3, microbatches=6)
    flat = make_params(cfg.model)
    _, ref, _ = _run(cfg, flat, "bf16", 2)
    probe = _gpu(cfg, flat, "bf16")
    slot = max(probe.stage_memory(s)[0] for s in range(cfg.stages))
    probe.close()
    plans = opl.normal_plans(cfg.stages, cfg.microbatches, True)
    swapped = 0
    for v in range(cfg.stages):
        for pi in (3, len(plans[v]) // 2, len(plans[v]) - 6):
            p, got, rec = _run(cfg, flat, "bf16", 2, inject=(0, v, pi), frc_retain_bytes=slot,
                               frc_swap_bytes=host_sets * slot)
            for (la, sa), (lb, sb) in zip(got, ref):
                assert la == lb, (v, pi)
                for w in sa:
                    assert np.array_equal(sa[w], sb[w]), (v, pi, w)
            swapped += rec.frc_swapped_mb
            # host slots per replica = swap bytes / that stage's saved-set size
            assert rec.frc_swapped_mb <= cfg.microbatches - 1
            p.close()
    assert swapped > 0


def test_frc_tile_grid_bitwise_and_node_stats():
    """FRC GEMMs on one-CTA-per-tile grids (default) vs persistent grids:
    identical results bit for bit; per-node accounting is consistent."""
    cfg = dataclasses.replace(get_config("C0"), stages=3, microbatches=6)
    flat = make_params(cfg.model)
    _, a, _ = _run(cfg, flat, "bf16", 2, frc_persistent=True)
    p, b, _ = _run(cfg, flat, "bf16", 2, timing=True)
    for (la, sa), (lb, sb) in zip(a, b):
        assert la == lb
        for w in sa:
            assert np.array_equal(sa[w], sb[w]), w
    stats = p.node_stats()
    assert len(stats) == cfg.stages
    for s in stats:
        assert s["n_fwd"] == cfg.microbatches and s["n_bwd"] == cfg.microbatches
        assert s["n_frc"] == cfg.microbatches
        assert 0 < s["busy_ms"] <= s["step_ms"] + 1e-3
        assert abs(s["busy_ms"] + s["bubble_ms"] - s["step_ms"]) < 1e-3
        assert -1e-3 <= s["frc_hidden_ms"] <= s["frc_ms"] + 1e-3
    p.close()


@pytest.mark.parametrize("lps", [[3, 1, 0], [0, 2, 2], [2, 1, 1]])
def test_custom_partition_matches_oracle(lps):
    """layers_per_stage (bb_opts): a head-only last stage and an
    embedding-only first stage (the cost-balanced partitions bench.py uses)
    give the oracle's loss and gradients, and a preemption of the head-only /
    embedding-only node recovers bit for bit."""
    c0 = get_config("C0")
    cfg = dataclasses.replace(c0, stages=3, microbatches=4)
    flat = make_params(cfg.model)
    p = _gpu(cfg, flat, "bf16", layers_per_stage=lps)
    ref = opipe.Pipeline(cfg, flat, rc=True, lr=LR, layers_per_stage=lps)
    want = opl.dump(cfg.stages, cfg.microbatches, True, opl.partition(cfg.model.n_layer, 3, lps),
                    opl.normal_plans(cfg.stages, cfg.microbatches, True))
    assert p.schedule_dump() == want
    tok, tgt = make_tokens(cfg, 0)
    s0 = _state0(ref)
    status, st = p.step(tok, tgt)
    _, ref_loss = ref.step(tok, tgt)
    _compare_step(cfg, p, ref, "bf16", st.loss, ref_loss, s0)
    base = {w: _flat_state(p, 3, w) for w in STATES}
    p.close()
    for victim, kw in ((0, {}), (2, {}),
                       # the automatic FRC budget and the host tier with an
                       # embedding-only stage (its saved sets are empty)
                       (1, dict(frc_retain_bytes=(1 << 64) - 1)),
                       (1, dict(frc_retain_bytes=1, frc_swap_bytes=1 << 20))):
        q = _gpu(cfg, flat, "bf16", layers_per_stage=lps, **kw)
        q.preempt(victim, 9)
        status, st = q.step(tok, tgt)
        assert status == "preempted"
        q.recover()
        for w, v in base.items():
            assert np.array_equal(_flat_state(q, 3, w), v), (victim, w)
        q.close()


def test_non_adjacent_second_preemption_bitwise():
    """SPEC S:537 / P:464: after a failover, a preemption of a node that is not
    adjacent to the dead one is a second, independent recovery. P=5 stages on
    one GPU: lose node 1 mid-step, run a failover step, lose node 3 (or 4) at
    several points, run the double-failover plan, rejoin both (LIFO): every
    step equals the failure-free run bit for bit; the dumps equal the
    oracle's; an adjacent loss is FATAL."""
    import paper_2204_12013_b200 as bb
    cfg = dataclasses.replace(get_config("C0"), model=dataclasses.replace(
        get_config("C0").model, n_layer=5), stages=5, microbatches=4)
    flat = make_params(cfg.model)
    _, ref, _ = _run(cfg, flat, "bf16", 6)
    for v2 in (3, 4):
        n2 = len(opl.failover_plans(5, 4, 1)[v2])
        for pi2 in (0, n2 // 2, n2):
            p = _gpu(cfg, flat, "bf16")
            oref = opipe.Pipeline(cfg, flat, rc=True, lr=LR)
            for t in range(6):
                tok, tgt = make_tokens(cfg, t)
                ev = {0: (1, 7), 2: (v2, pi2)}.get(t)
                if t == 4 or t == 5:
                    p.rejoin()
                    oref.rejoin()
                if ev is not None:
                    p.preempt(*ev)
                    oref.preempt(*ev)
                status, st = p.step(tok, tgt)
                if status == "preempted":
                    loss = p.recover().loss
                    oref.step(tok, tgt)
                    oref.recover()
                    if t == 2:
                        with pytest.raises(bb.BambooError) as e:
                            p.preempt(2, 0)     # adjacent to node 3 / shadow of 3
                        assert e.value.status == bb.BB_E_FATAL or v2 == 4
                else:
                    loss = st.loss
                    oref.step(tok, tgt)
                assert loss == ref[t][0], (v2, pi2, t)
                for w in STATES:
                    assert np.array_equal(_flat_state(p, cfg.stages, w), ref[t][1][w]), (t, w)
                assert p.schedule_dump() == oref.dump(), (v2, pi2, t)
            p.close()


def test_lflb_recovery_bitwise_and_plans():
    """LFLB: replicas in sync, no FRC in the normal step; on a
    failure the shadow recomputes the victim's forward and backward for the
    step. Same results as the failure-free EFLB run, bit for bit; plan and
    recovery dumps equal the oracle's."""
    cfg = dataclasses.replace(get_config("C0"), stages=3, microbatches=4)
    flat = make_params(cfg.model)
    _, ref, _ = _run(cfg, flat, "bf16", 2)
    p0 = _gpu(cfg, flat, "bf16", rc="lflb")
    assert p0.schedule_dump() == opl.dump(3, 4, "lflb", opl.partition(4, 3),
                                          opl.normal_plans(3, 4, "lflb"))
    p0.close()
    plans = opl.normal_plans(3, 4, "lflb")
    for v in range(3):
        for pi in (2, len(plans[v]) // 2, len(plans[v]) - 3, len(plans[v])):
            p, got, rec = _run(cfg, flat, "bf16", 2, inject=(0, v, pi), rc="lflb")
            assert p.recovery_dump() == opl.recovery_dump(3, 4, v, pi, rc="lflb")
            assert rec.frc_done_mb == 0
            for t, ((la, sa), (lb, sb)) in enumerate(zip(got, ref)):
                if t == 0 and v == 2 and rec.commit:
                    assert np.isnan(la)     # the loss left with the last stage
                else:
                    assert la == lb, (v, pi, t)
                for w in sa:
                    assert np.array_equal(sa[w], sb[w]), (v, pi, w)
            p.close()


def test_zipf_tokens_embedding_backward_matches_oracle():
    """Zipf(1.1) tokens: many repeated ids per micro-batch
    stress the device-built token CSR of the deterministic embedding
    backward; gradients match the oracle and two runs are bit-identical."""
    cfg = get_config("C0")
    flat = make_params(cfg.model)
    tok, tgt = make_tokens(cfg, 0, zipf=True)
    assert len(np.unique(tok[:cfg.micro_batch])) < tok[:cfg.micro_batch].size * 3 // 4
    outs = []
    for _ in range(2):
        p = _gpu(cfg, flat, "bf16")
        ref = opipe.Pipeline(cfg, flat, rc=True, lr=LR)
        s0 = _state0(ref)
        _, st = p.step(tok, tgt)
        _, rl = ref.step(tok, tgt)
        _compare_step(cfg, p, ref, "bf16", st.loss, rl, s0)
        outs.append(_flat_state(p, cfg.stages, "grads"))
        p.close()
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("P", [2, 3, 4])
def test_efeb_eager_brc_bitwise(P):
    """EFEB: every node runs its replica stage's backward
    eagerly on the FRC stream from the duplicate gradient of node s+2, so the
    replica's gradient and state equal the primary's with no replica sync.
    Results equal the failure-free EFLB run bit for bit; a preemption at
    several points of every victim recovers bit for bit with plans equal to
    the oracle's, and the recovery reuses the eager BRC (few or no
    re-computed backwards)."""
    cfg = dataclasses.replace(get_config("C0"), stages=P, microbatches=4)
    flat = make_params(cfg.model)
    _, ref, _ = _run(cfg, flat, "bf16", 2)
    p, got, _ = _run(cfg, flat, "bf16", 2, rc="efeb")
    assert p.schedule_dump() == opl.dump(P, 4, "efeb", opl.partition(4, P),
                                         opl.normal_plans(P, 4, "efeb"))
    for s in range(P):
        for w in STATES:
            assert np.array_equal(p.read_state(s, w), p.read_state(s, w, replica=True)), (s, w)
    p.close()
    for (la, sa), (lb, sb) in zip(got, ref):
        assert la == lb
        for w in sa:
            assert np.array_equal(sa[w], sb[w]), w
    plans = opl.normal_plans(P, 4, "efeb")
    for v in range(P):
        n = len(plans[v])
        for pi in sorted({1, n // 3, n // 2, (2 * n) // 3, n}):
            q, got2, rec = _run(cfg, flat, "bf16", 2, inject=(0, v, pi), rc="efeb")
            assert q.recovery_dump() == opl.recovery_dump(P, 4, v, pi, rc="efeb"), (v, pi)
            for (la, sa), (lb, sb) in zip(got2, ref):
                assert la == lb, (v, pi)
                for w in sa:
                    assert np.array_equal(sa[w], sb[w]), (v, pi, w)
            q.close()
