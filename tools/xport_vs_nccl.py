"""The library's inter-process transport vs NCCL P2P: one-way
time per message of a 2-process ping-pong, same sizes (C1 / C3 activation =
the pipeline's per-micro-batch message), one process per GPU.

    torchrun --nproc-per-node 2 tools/xport_vs_nccl.py > out.json
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2204_12013_b200 as bb  # noqa: E402

SIZES = {"64KiB": 64 << 10, "1MiB": 1 << 20, "C1 act 12MiB": 8 * 1024 * 768 * 2,
         "C3 act 12.5MiB": 4 * 1024 * 1600 * 2, "C2 act 16MiB": 16 * 512 * 1024 * 2}
ITERS = 200


def main():
    rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    out = {"gpus": torch.cuda.device_count(), "iters": ITERS, "nccl_us": {}, "xport_us": {}}
    for name, n in SIZES.items():
        t = torch.zeros(n // 2, dtype=torch.bfloat16, device="cuda")
        for _ in range(10):   # warm-up
            if rank == 0:
                dist.send(t, 1)
                dist.recv(t, 1)
            else:
                dist.recv(t, 0)
                dist.send(t, 0)
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(ITERS):
            if rank == 0:
                dist.send(t, 1)
                dist.recv(t, 1)
            else:
                dist.recv(t, 0)
                dist.send(t, 0)
        torch.cuda.synchronize()
        out["nccl_us"][name] = round(1e6 * (time.perf_counter() - t0) / (2 * ITERS), 2)
        obj = [bb.session_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        bb.xport_pingpong(rank, 2, dev, obj[0], n, 10)
        obj = [bb.session_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        out["xport_us"][name] = round(bb.xport_pingpong(rank, 2, dev, obj[0], n, ITERS), 2)
        dist.barrier()
    if rank == 0:
        out["GBps_at_C3_act"] = {
            k: round(SIZES["C3 act 12.5MiB"] / (out[k]["C3 act 12.5MiB"] * 1e-6) / 1e9, 1)
            for k in ("nccl_us", "xport_us")}
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
