"""Time single kernels through the C ABI's bb_op_* entry points at the config
shapes (CUDA events, warm-up, median of repeats). Usage: op_bench.py C1|C3"""
import os, sys
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2204_12013_b200 as bb
from synth import get_config

cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "C1")
m = cfg.model
R, H, F, V, S, nh = cfg.micro_batch * m.seq_len, m.d_model, m.d_ff, m.vocab, m.seq_len, m.n_head
B = cfg.micro_batch
dev = "cuda"
bf = torch.bfloat16


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def rnd(*s, dt=bf):
    return (torch.randn(*s, device=dev) * 0.5).to(dt)


rows = []
x, g, bb_ = rnd(R, H), rnd(H), rnd(H)
y = torch.empty(R, H, device=dev, dtype=bf)
mean = torch.empty(R, device=dev); rstd = torch.empty(R, device=dev)
us = t(lambda: bb.op_layernorm_fwd("bf16", R, H, x.data_ptr(), g.data_ptr(), bb_.data_ptr(), y.data_ptr(), mean.data_ptr(), rstd.data_ptr()))
rows.append(("layernorm_fwd", us, 2 * R * H * 2 / us / 1e3, "GB/s"))
dy = rnd(R, H, dt=torch.float32); dres = rnd(R, H, dt=torch.float32)
dx = torch.empty(R, H, device=dev, dtype=bf); dg = torch.zeros(H, device=dev); db = torch.zeros(H, device=dev)
us = t(lambda: bb.op_layernorm_bwd("bf16", R, H, dy.data_ptr(), x.data_ptr(), mean.data_ptr(), rstd.data_ptr(), g.data_ptr(), dres.data_ptr(), dx.data_ptr(), dg.data_ptr(), db.data_ptr()))
rows.append(("layernorm_bwd(+dg,db)", us, R * H * (4 + 2 + 4 + 2) / us / 1e3, "GB/s"))
qkv = rnd(R, 3 * H); o = torch.empty(R, H, device=dev, dtype=bf); lse = torch.empty(B, nh, S, device=dev)
att_fl = 4 * B * nh * S * S * (H // nh) * (0.5 if m.causal else 1.0)
us = t(lambda: bb.op_attention_fwd("bf16", B, S, H, nh, m.causal, qkv.data_ptr(), o.data_ptr(), lse.data_ptr()))
rows.append(("attention_fwd", us, att_fl / us / 1e6, "TFLOP/s"))
do = rnd(R, H); dqkv = torch.empty(R, 3 * H, device=dev, dtype=bf)
us = t(lambda: bb.op_attention_bwd("bf16", B, S, H, nh, m.causal, qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), do.data_ptr(), dqkv.data_ptr()))
rows.append(("attention_bwd", us, 2.5 * att_fl / us / 1e6, "TFLOP/s"))
for name, (M_, N_, K_, amn, bmn, epi) in {
        "gemm qkv fwd": (R, 3 * H, H, 0, 0, 1), "gemm proj fwd": (R, H, H, 0, 0, 2),
        "gemm fc1 fwd": (R, F, H, 0, 0, 3), "gemm fc2 fwd": (R, H, F, 0, 0, 2),
        "gemm head fwd": (R, V, H, 0, 0, 0), "gemm fc2 dX(gelu')": (R, F, H, 0, 1, 4),
        "gemm fc1 dX": (R, H, F, 0, 1, 6), "gemm fc2 dW": (H, F, R, 1, 1, 5),
        "gemm proj dW": (H, H, R, 1, 1, 5), "gemm head dW": (V, H, R, 1, 1, 5)}.items():
    A = rnd(K_, M_) if amn else rnd(M_, K_)
    Bm = rnd(K_, N_) if bmn else rnd(N_, K_)
    f32 = epi in (5, 6)
    C = torch.zeros(M_, N_, device=dev, dtype=torch.float32 if f32 else bf)
    bias = rnd(N_); res = rnd(M_, N_); aux = rnd(M_, N_)
    us = t(lambda: bb.op_gemm("bf16", 0, M_, N_, K_, A.data_ptr(), M_ if amn else K_, amn, Bm.data_ptr(), N_ if bmn else K_, bmn, epi, C.data_ptr(), N_, bias.data_ptr(), res.data_ptr(), aux.data_ptr()))
    rows.append((f"{name} {M_}x{N_}x{K_}", us, 2 * M_ * N_ * K_ / us / 1e6, "TFLOP/s"))
logits = rnd(R, V); tg = torch.randint(0, V, (R,), device=dev, dtype=torch.int32); lr_ = torch.empty(R, device=dev)
us = t(lambda: bb.op_cross_entropy("bf16", R, V, logits.data_ptr(), tg.data_ptr(), R * 4, lr_.data_ptr()))
rows.append(("cross_entropy", us, 3 * R * V * 2 / us / 1e3, "GB/s"))
print(f"{cfg.name}: R={R} H={H} F={F} V={V} S={S} heads={nh}")
for n, us, rate, unit in rows:
    print(f"{n:40s} {us:9.1f} us  {rate:8.1f} {unit}")
