"""Time one bf16 GEMM shape through bb_op_gemm under each tile kind
(BB_GEMM_TILE = 128 / 256 / pair, one subprocess each).

    python tools/gemm_probe.py M N K [a_mn b_mn epi]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import sys, torch
sys.path.insert(0, %r)
import paper_2204_12013_b200 as bb
M, N, K, amn, bmn, epi = %s
bf = torch.bfloat16
A = (torch.randn(K, M, device="cuda") if amn else torch.randn(M, K, device="cuda")).to(bf)
B = (torch.randn(K, N, device="cuda") if bmn else torch.randn(N, K, device="cuda")).to(bf)
f32 = epi in (5, 6)
C = torch.zeros(M, N, device="cuda", dtype=torch.float32 if f32 else bf)
aux = torch.zeros(M, N, device="cuda", dtype=bf)
bias = torch.zeros(N, device="cuda", dtype=bf)
res = torch.zeros(M, N, device="cuda", dtype=bf)
f = lambda: bb.op_gemm("bf16", 0, M, N, K, A.data_ptr(), M if amn else K, amn, B.data_ptr(),
                       N if bmn else K, bmn, epi, C.data_ptr(), N, bias.data_ptr(), res.data_ptr(),
                       aux.data_ptr())
for _ in range(5): f()
torch.cuda.synchronize()
ts = []
for _ in range(30):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); f(); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
ts.sort()
us = ts[len(ts) // 2]
# back-to-back batch: device time per launch with the queue kept full
import time
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda._sleep(20_000_000)   # ~10 ms of GPU spin so the host runs ahead
a.record()
h0 = time.perf_counter()
for _ in range(50): f()
h1 = time.perf_counter()
b.record(); torch.cuda.synchronize()
bus = a.elapsed_time(b) * 1e3 / 50
print(f"{M}x{N}x{K} a_mn={amn} b_mn={bmn} epi={epi}: {us:8.1f} us single, {bus:8.1f} us batched"
      f" {2*M*N*K/bus/1e6:7.1f} TF/s, host {1e6*(h1-h0)/50:5.1f} us/launch")
'''


def main():
    a = [int(x) for x in sys.argv[1:]]
    M, N, K = a[:3]
    amn, bmn, epi = (a[3:] + [0, 0, 0])[:3] if len(a) > 3 else (0, 0, 0)
    tiles = os.environ.get("TILES", "128,256,pair").split(",")
    for tile in tiles:
        env = dict(os.environ, BB_GEMM_TILE=tile)
        r = subprocess.run([sys.executable, "-c", CHILD % (ROOT, (M, N, K, amn, bmn, epi))],
                           env=env, capture_output=True, text=True)
        print(f"tile {tile:5s}", (r.stdout.strip() or r.stderr.strip()[-500:]), flush=True)


if __name__ == "__main__":
    main()
