"""Host-side parity (no GPU): the C++ controller in libbamboo.so must emit
byte-identical plan / failover / recovery dumps to the oracle (SURVEY.md §8(b)
"schedule and stage assignment bit-exact"), and the library must export every
entry point declared in include/bamboo.h."""
import os
import random
import re

import pytest

from oracle import plan as pl
from synth import get_config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
bbl = pytest.importorskip("paper_2204_12013_b200._lib")


def _lib_or_skip():
    if not os.path.exists(bbl.LIB_PATH):
        pytest.skip("libbamboo.so not built")
    return bbl.lib()


def test_exports_every_header_symbol():
    lib = _lib_or_skip()
    hdr = open(os.path.join(ROOT, "include", "bamboo.h")).read()
    names = sorted(set(re.findall(r"^(?:bb_status|void)\s+\*?(bb_[a-z0-9_]+)\s*\(", hdr, re.M)))
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert set(bbl.EXPORTED) <= set(names)


def _oracle_normal(cfg, P, M, rc, world_size=1):
    per = -(-P // world_size)
    dev = {n: min(n // per, world_size - 1) for n in range(P)}
    return pl.dump(P, M, rc, pl.partition(cfg.model.n_layer, P), pl.normal_plans(P, M, rc),
                   device=dev)


@pytest.mark.parametrize("name", ["C0", "C1", "C2", "C3"])
@pytest.mark.parametrize("rc", [True, False])
def test_normal_plan_dump_matches_oracle(name, rc):
    _lib_or_skip()
    cfg = get_config(name)
    P, M = cfg.stages, cfg.microbatches
    for ws in (1, 2, P):
        got = bbl.plan_dump(cfg.model, P, M, rc=rc, world_size=ws)
        assert got == _oracle_normal(cfg, P, M, rc, ws)


def test_failover_and_recovery_dumps_match_oracle():
    _lib_or_skip()
    r = random.Random(3)
    cfg = get_config("C3")   # 48 layers: any P <= 8 is valid
    cases = [(2, 4), (8, 32), (4, 8), (8, 16)] + [(r.randint(2, 8), r.randint(1, 32))
                                                 for _ in range(12)]
    for P, M in cases:
        plans = pl.normal_plans(P, M, True)
        for v in range(P):
            host, rep = pl.failover_topology(P, v)
            want = pl.dump(P, M, True, pl.partition(48, P), pl.failover_plans(P, M, v), host, rep,
                           mode="failover", victim=v)
            assert bbl.plan_dump(cfg.model, P, M, victim=v, at_instr=-1) == want
            pis = {0, len(plans[v]), len(plans[v]) // 2} | {r.randint(0, len(plans[v]))
                                                             for _ in range(3)}
            for pi in sorted(pis):
                assert bbl.plan_dump(cfg.model, P, M, victim=v, at_instr=pi) == \
                    pl.recovery_dump(P, M, v, pi), (P, M, v, pi)


def test_invalid_configs_rejected():
    _lib_or_skip()
    cfg = get_config("C0")
    with pytest.raises(bbl.BambooError):
        bbl.plan_dump(cfg.model, 5, 4)              # stages > n_layer
    with pytest.raises(bbl.BambooError):
        bbl.plan_dump(cfg.model, 1, 4, victim=0)    # no replica without RC partner


def test_cpp_failover_goldens():
    """The library's merge reproduces the hand-derived P=3 goldens
    (tests/golden/p3_m2_failover_v*.txt)."""
    import os
    gold = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    m = dict(n_layer=3, d_model=64, n_head=2, d_ff=256, vocab=128, seq_len=32, causal=1)
    for v in (0, 1):
        text = bbl.plan_dump(m, 3, 2, victim=v, micro_batch=1)
        lines = "".join(l + "\n" for l in text.splitlines() if not l.startswith("#"))
        assert lines == open(os.path.join(gold, f"p3_m2_failover_v{v}.txt")).read(), v


def test_cpp_lflb_plans_match_oracle():
    r = random.Random(9)
    m = dict(n_layer=6, d_model=64, n_head=2, d_ff=256, vocab=128, seq_len=32, causal=1)
    for _ in range(20):
        P, M = r.randint(2, 6), r.randint(1, 7)
        got = bbl.plan_dump(m, P, M, rc="lflb", micro_batch=1)
        want = pl.dump(P, M, "lflb", pl.partition(6, P), pl.normal_plans(P, M, "lflb"))
        assert got == want, (P, M)
        v = r.randrange(P)
        n = len(pl.normal_plans(P, M, "lflb")[v])
        pi = r.randint(0, n)
        assert bbl.plan_dump(m, P, M, victim=v, at_instr=pi, rc="lflb", micro_batch=1) == \
            pl.recovery_dump(P, M, v, pi, rc="lflb"), (P, M, v, pi)


@pytest.mark.parametrize("mode", ["eflb", "lflb", "efeb"])
def test_cpp_recovery_matches_oracle_every_point(mode):
    """The library's recovery planner (plan.cpp, written from the rules with a
    dependency-graph merge) and the oracle's (co-simulating merge) agree on
    the cut and continuation text of every injection point of every victim,
    for P = 2..5 and several M, in every RC mode; and on the static failover
    plans."""
    m = dict(n_layer=6, d_model=64, n_head=2, d_ff=256, vocab=128, seq_len=32, causal=1)
    for P in (2, 3, 4, 5):
        for M in (1, 2, 3, 6):
            plans = pl.normal_plans(P, M, mode)
            assert bbl.plan_dump(m, P, M, rc=mode, micro_batch=1) == \
                pl.dump(P, M, mode, pl.partition(6, P), plans)
            for v in range(P):
                host, rep = pl.failover_topology(P, v)
                assert bbl.plan_dump(m, P, M, victim=v, rc=mode, micro_batch=1) == \
                    pl.dump(P, M, mode, pl.partition(6, P), pl.failover_plans(P, M, v, plans),
                            host, rep, mode="failover", victim=v), (P, M, v)
                for pi in range(len(plans[v]) + 1):
                    assert bbl.plan_dump(m, P, M, victim=v, at_instr=pi, rc=mode,
                                         micro_batch=1) == \
                        pl.recovery_dump(P, M, v, pi, rc=mode), (P, M, v, pi)


@pytest.mark.parametrize("mode", ["none", "eflb", "lflb", "efeb"])
def test_cpp_dp_plans_match_oracle_every_point(mode):
    """D > 1 data-parallel pipelines: normal dumps (with the
    default rank layout over 1, 2 and D*P processes), failover dumps of every
    node and the cut + continuation of every injection point agree with the
    oracle's, including the other pipelines' re-sent all-reduce
    contributions."""
    m = dict(n_layer=6, d_model=64, n_head=2, d_ff=256, vocab=128, seq_len=32, causal=1)
    for P, M, D in ((2, 1, 2), (2, 2, 2), (3, 2, 2), (2, 3, 3), (4, 2, 2)):
        plans = pl.normal_plans(P, M, mode, D)
        host, rep = pl.normal_topology(P, D)
        if mode == "none":
            rep = {g: None for g in host}
        for ws in (1, 2, D * P):
            per = -(-(D * P) // ws)
            dev = {n: min(n // per, ws - 1) for n in range(D * P)}
            assert bbl.plan_dump(m, P, M, rc=mode, micro_batch=1, pipelines=D, world_size=ws) == \
                pl.dump(P, M, mode, pl.partition(6, P), plans, host, rep, dev), (P, M, D, ws)
        if mode == "none":
            continue
        for v in range(D * P):
            fh, fr = pl.failover_topology(P, v, D)
            assert bbl.plan_dump(m, P, M, victim=v, rc=mode, micro_batch=1, pipelines=D) == \
                pl.dump(P, M, mode, pl.partition(6, P), pl.failover_plans(P, M, v, plans),
                        fh, fr, mode="failover", victim=v), (P, M, D, v)
            for pi in range(len(plans[v]) + 1):
                assert bbl.plan_dump(m, P, M, victim=v, at_instr=pi, rc=mode, micro_batch=1,
                                     pipelines=D) == \
                    pl.recovery_dump(P, M, v, pi, rc=mode, D=D), (P, M, D, v, pi)


def test_dp_recovery_golden():
    """Hand-derived D=2 recovery (tests/golden/README.md): both planners."""
    gold = open(os.path.join(ROOT, "tests", "golden", "dp2_p2_m1_v3_pi7_recovery.txt")).read()
    assert pl.recovery_dump(2, 1, 3, 7, "eflb", D=2) == gold
    _lib_or_skip()
    m = dict(n_layer=2, d_model=64, n_head=2, d_ff=256, vocab=128, seq_len=32, causal=1)
    assert bbl.plan_dump(m, 2, 1, victim=3, at_instr=7, micro_batch=1, pipelines=2) == gold
