"""World-size-2 host-side checks of the multi-process path on CPU (gloo; no
GPU). Every rank computes the plans, the injection cut and the recovery /
failover continuation independently from the static plans (no coordinator,
DESIGN.md §2 Q12/Q14); these must agree byte for byte across ranks and with
the oracle, for contiguous and interleaved node->rank maps."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import plan as opl
from synth import get_config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, ws, port, node_rank, q):
    import sys
    sys.path.insert(0, ROOT)
    import paper_2204_12013_b200 as bb
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    cfg = get_config("C0")
    P, M = 4, 6
    m = dict(n_layer=4, d_model=64, n_head=2, d_ff=256, vocab=128, seq_len=32, causal=1)
    kw = dict(micro_batch=2, world_rank=rank, world_size=ws, node_rank=node_rank)
    texts = [bb.plan_dump(m, P, M, **kw)]
    for v in range(P):
        texts.append(bb.plan_dump(m, P, M, victim=v, **kw))
        n = len(opl.normal_plans(P, M, True)[v])
        for pi in (0, n // 3, n // 2, n):
            texts.append(bb.plan_dump(m, P, M, victim=v, at_instr=pi, **kw))
    got = [None] * ws
    dist.all_gather_object(got, texts)
    if rank == 0:
        q.put(got)
    dist.barrier()
    dist.destroy_process_group()
    del cfg


@pytest.mark.parametrize("node_rank", [[0, 0, 1, 1], [0, 1, 0, 1]])
def test_ranks_agree_on_plans_cuts_and_recovery(node_rank):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, node_rank, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = q.get(timeout=300)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got[0] == got[1]
    P, M = 4, 6
    texts = got[0]
    dev = {n: node_rank[n] for n in range(P)}
    assert texts[0] == opl.dump(P, M, True, opl.partition(4, P), opl.normal_plans(P, M, True),
                                device=dev)
    i = 1
    for v in range(P):
        host, rep = opl.failover_topology(P, v)
        assert texts[i] == opl.dump(P, M, True, opl.partition(4, P), opl.failover_plans(P, M, v),
                                    host, rep, device=dev, mode="failover", victim=v)
        i += 1
        n = len(opl.normal_plans(P, M, True)[v])
        for pi in (0, n // 3, n // 2, n):
            assert texts[i] == opl.recovery_dump(P, M, v, pi), (v, pi)
            i += 1
