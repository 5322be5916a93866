"""Every GEMM shape of a config's training step once, through the C ABI's
single-op entry point, after one warm-up round of all of them (for
`ncu --set full -k regex:gemm_tc --launch-skip <shapes>`: a full-set capture
per shape with a small device footprint). Prints the shape list.

    python tools/gemm_shapes.py C3
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2204_12013_b200 as bb  # noqa: E402
from synth import get_config  # noqa: E402

cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "C3")
m = cfg.model
R, H, F, V = cfg.micro_batch * m.seq_len, m.d_model, m.d_ff, m.vocab
dev, bf = "cuda", torch.bfloat16
# name: (M, N, K, a_mn, b_mn, epilogue) — forward, input-gradient, weight-gradient
SHAPES = {
    "qkv fwd": (R, 3 * H, H, 0, 0, 1), "proj fwd": (R, H, H, 0, 0, 2),
    "fc1 fwd": (R, F, H, 0, 0, 3), "fc2 fwd": (R, H, F, 0, 0, 2), "head fwd": (R, V, H, 0, 0, 0),
    "qkv dX": (R, H, 3 * H, 0, 1, 6), "proj dX": (R, H, H, 0, 1, 6),
    "fc1 dX": (R, H, F, 0, 1, 6), "fc2 dX(gelu')": (R, F, H, 0, 1, 4),
    "head dX": (R, H, V, 0, 1, 6),
    "qkv dW": (3 * H, H, R, 1, 1, 5), "proj dW": (H, H, R, 1, 1, 5),
    "fc1 dW": (F, H, R, 1, 1, 5), "fc2 dW": (H, F, R, 1, 1, 5), "head dW": (V, H, R, 1, 1, 5),
}


def run(shape):
    M_, N_, K_, amn, bmn, epi = shape
    g = torch.Generator(device=dev).manual_seed(0)
    A = (torch.randn(K_, M_, device=dev, generator=g) if amn else
         torch.randn(M_, K_, device=dev, generator=g)).to(bf)
    B = (torch.randn(K_, N_, device=dev, generator=g) if bmn else
         torch.randn(N_, K_, device=dev, generator=g)).to(bf)
    f32 = epi in (5, 6)
    C = torch.zeros(M_, N_, device=dev, dtype=torch.float32 if f32 else bf)
    bias = torch.zeros(N_, device=dev, dtype=bf)
    res = torch.zeros(M_, N_, device=dev, dtype=bf)
    aux = torch.zeros(M_, N_, device=dev, dtype=bf)
    bb.op_gemm("bf16", 0, M_, N_, K_, A.data_ptr(), M_ if amn else K_, amn, B.data_ptr(),
               N_ if bmn else K_, bmn, epi, C.data_ptr(), N_, bias.data_ptr(), res.data_ptr(),
               aux.data_ptr())
    torch.cuda.synchronize()


for s in SHAPES.values():   # warm-up round (skipped by ncu --launch-skip)
    run(s)
for name, s in SHAPES.items():
    run(s)
    print(name, s, flush=True)
