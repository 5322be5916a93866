"""Pins for oracle/plan.py: SPEC examples, analytic 1F1B duration, the Fig-6
bubble, the hand-derived Appendix-B goldens and the merge property suite."""
import os
import random

import pytest

from oracle import plan as pl

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def kinds(seq):
    return [(i.kind, i.mb) for i in seq]


def test_partition_even_remainder_last():
    # P:517 "more layers are placed on the last few stages"
    assert pl.partition(4, 2) == [(0, 2), (3, 5)]
    assert pl.partition(12, 4) == [(0, 3), (4, 6), (7, 9), (10, 13)]
    r = pl.partition(10, 4)   # 2,2,3,3 blocks
    assert [b - a + 1 for a, b in r] == [3, 2, 3, 4]
    assert pl.partition(48, 8)[0] == (0, 6) and pl.partition(48, 8)[-1] == (43, 49)
    with pytest.raises(pl.PlanError):
        pl.partition(3, 4)     # P > layer count is invalid


def test_spec_p1_serial():
    # P=1, M=2 -> F0 B0 F1 B1 (then the update; D=1 has no all-reduce)
    seq = pl.stage_plan(0, 1, 2, False)
    assert kinds(seq) == [("LOAD_INPUTS", None), ("FWD", 0), ("BWD", 0), ("FWD", 1), ("BWD", 1),
                          ("APPLY", None)]


def test_rc_needs_two_stages():
    with pytest.raises(pl.PlanError):
        pl.stage_plan(0, 1, 4, True)


def _inflight(seq):
    cur = peak = 0
    for i in seq:
        if i.kind == "FWD":
            cur += 1
        elif i.kind == "BWD":
            cur -= 1
        peak = max(peak, cur)
    return peak


@pytest.mark.parametrize("P,M", [(4, 4), (4, 8), (3, 5), (5, 2)])
def test_1f1b_structure(P, M):
    plans = pl.normal_plans(P, M, False)
    last = [i.kind for i in plans[P - 1] if i.kind in ("FWD", "BWD")]
    assert last == ["FWD", "BWD"] * M
    peaks = [_inflight(plans[s]) for s in range(P)]
    assert all(a >= b for a, b in zip(peaks, peaks[1:]))
    assert peaks == [min(M, P - s) for s in range(P)]
    for s in range(P):
        fw = sorted(i.mb for i in plans[s] if i.kind == "FWD")
        bw = [i.mb for i in plans[s] if i.kind == "BWD"]
        assert fw == list(range(M)) and bw == list(range(M))   # S:148, ascending BWD
    pl.lockstep(plans)      # dependency soundness (FIFO asserts inside)


@pytest.mark.parametrize("P", range(1, 7))
@pytest.mark.parametrize("M", range(1, 9))
def test_1f1b_analytic_duration(P, M):
    # S:191 / S:530: uniform stages, zero comm: (M + P - 1)(f + b)
    f, b = 1.0, 2.0
    plans = pl.normal_plans(P, M, False)
    ends, _ = pl.simulate_times(plans, P, [f] * P, [b] * P)
    assert max(ends.values()) == pytest.approx((M + P - 1) * (f + b))


def test_fig6_bubble():
    # P:488 fig:instr-group: forward on node i and i+1 take t and 1.2t (b = 2f):
    # node i waits 0.6t at the barrier in every steady-state cycle.
    t = 1.0
    P, M = 2, 12
    plans = pl.normal_plans(P, M, False)
    ends, tl = pl.simulate_times(plans, P, [t, 1.2 * t], [2 * t, 2.4 * t])
    busy = [(s, e) for k, mb, s, e in tl[0] if k in ("FWD", "BWD")]
    gaps = [b[0] - a[1] for a, b in zip(busy, busy[1:])]
    steady = [g for g in gaps[3:-3] if g > 1e-12]
    assert steady and all(g == pytest.approx(0.6 * t) for g in steady)


def test_golden_c0_normal_plan():
    P, M = 2, 4
    text = pl.dump(P, M, True, pl.partition(4, P), pl.normal_plans(P, M, True))
    assert text == open(os.path.join(GOLD, "c0_plan_eflb.txt")).read()


def test_golden_c0_failover_plan():
    P, M, v = 2, 4, 1
    host, rep = pl.failover_topology(P, v)
    text = pl.dump(P, M, True, pl.partition(4, P), pl.failover_plans(P, M, v), host, rep,
                   mode="failover", victim=v)
    assert text == open(os.path.join(GOLD, "c0_plan_failover_v1.txt")).read()


def test_frc_is_intra_node_and_after_own_forward():
    # FRC creates only intra-node dependencies; FRC_FWD(k) on s<P-1
    # follows FWD(k); on P-1 it needs only inputs.
    for P in (2, 3, 5):
        plans = pl.normal_plans(P, 6, True)
        for s in range(P):
            seen = set()
            for i in plans[s]:
                if i.kind == "FWD":
                    seen.add(i.mb)
                if i.kind == "FRC_FWD":
                    assert i.stage == (s + 1) % P
                    if s < P - 1:
                        assert i.mb in seen
        pl.lockstep(plans)


def _check_failover(P, M, v, plans_new):
    u = (v - 1) % P
    assert v not in plans_new
    for n, seq in plans_new.items():
        for i in seq:
            assert i.peer != v                     # rerouted, nothing talks to v
            if n == u:
                assert not (i.kind in pl.COMMS and i.peer == u)
    # topological: the whole failover plan set runs to completion in lockstep
    pcs, ch = pl.lockstep(plans_new)
    assert all(pcs[n] == len(plans_new[n]) for n in plans_new)
    assert all(len(q) == 0 for q in ch.values())
    # every stage still does M forwards and M backwards, in ascending order
    for X in range(P):
        host = u if X == v else X
        fw = [i.mb for i in plans_new[host] if i.kind == "FWD" and i.stage == X]
        bw = [i.mb for i in plans_new[host] if i.kind == "BWD" and i.stage == X]
        assert fw == list(range(M)) and bw == list(range(M))
    # S:535 merge checks on the shadow's list. Provenance is read off the
    # stage field (the victim's work acts for stage v, the shadow's own for
    # u or none), so the two sequences are recovered without the merge's
    # internals; readiness here is data readiness only (local input keys),
    # so RECV heads (arrival-dependent) are not judged.
    _check_merge_rules(P, M, u, v, plans_new[u])


def _check_merge_rules(P, M, u, v, seq):
    side = lambda ins: 0 if ins.stage == v else 1          # 0 = victim's, 1 = shadow's
    A = [i for i in seq if side(i) == 1]
    B = [i for i in seq if side(i) == 0]
    heads = {0: 0, 1: 0}
    lists = {0: B, 1: A}
    avail = set()
    data_ready = lambda ins: all(k in avail for k in pl.inputs_of(ins, P))
    for ins in seq:
        s = side(ins)
        assert all(k in avail for k in pl.inputs_of(ins, P)) or ins.kind in pl.RECVS
        o = 1 - s
        other = lists[o][heads[o]] if heads[o] < len(lists[o]) else None
        if other is not None and other.kind not in pl.RECVS and data_ready(other):
            if ins.kind not in pl.COMMS:
                # rule 1: no ready communication left waiting behind a computation
                assert other.kind not in pl.SENDS, ("rule 1", ins, other)
                # rule 4: no ready backward left waiting behind a forward
                assert not (ins.kind == pl.FWD and other.kind == pl.BWD), ("rule 4", ins, other)
            elif s == 1:
                # rule 3: the victim's external communication goes first
                assert other.kind not in pl.SENDS, ("rule 3", ins, other)
        heads[s] += 1
        avail.update(pl.outputs_of(ins, P, M))


def test_failover_property_suite():
    # 1000 random adjacent victim/shadow pairs, P <= 5, M <= 6
    r = random.Random(7)
    for _ in range(1000):
        P = r.randint(2, 5)
        M = r.randint(1, 6)
        v = r.randrange(P)
        _check_failover(P, M, v, pl.failover_plans(P, M, v))


def test_recovery_property_suite():
    # every injection point of every victim: the continuation completes and
    # runs the victim's backward for every micro-batch (Q2) unless committed
    for P in (2, 3, 4):
        for M in (1, 3, 5):
            plans = pl.normal_plans(P, M, True)
            for v in range(P):
                for pi in range(len(plans[v]) + 1):
                    pcs, ch = pl.cut(plans, v, pi)
                    new, info = pl.recovery_plans(plans, P, M, v, pcs, ch)
                    pcs2, ch2 = pl.lockstep(new, {n: 0 for n in new}, ch)
                    assert all(pcs2[n] == len(new[n]) for n in new), (P, M, v, pi)
                    assert all(len(q) == 0 for q in ch2.values())
                    if not info["commit"]:
                        assert info["brc_mb"] == list(range(M))


def test_failover_goldens_exercise_merge_rules_1_3_4():
    """P=3, M=2 failover plans derived by hand from the four rules of
    P:538-545 (tests/golden/README.md walks the derivation): v=1 (shadow 0,
    rule 1: RECV_GRAD / REPLICA_SEND before ready computations) and v=0
    (shadow 2 = last stage, the wrap case: rule 3 puts the victim's
    RECV_GRAD ahead of the shadow's ready RECV_ACT / REPLICA_SEND, rule 4
    BWD before a ready FWD)."""
    for v in (0, 1):
        want = open(os.path.join(GOLD, f"p3_m2_failover_v{v}.txt")).read()
        assert pl.dump_lines(pl.failover_plans(3, 2, v)) == want, v
