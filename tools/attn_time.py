"""Attention forward + backward at a config's shape, a few times (for ncu
launch lists: `ncu --metrics gpu__time_duration.sum -k regex:fa_|dq_reduce`).

    python tools/attn_time.py C3 [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2204_12013_b200 as bb  # noqa: E402
from synth import get_config  # noqa: E402

cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "C3")
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
m = cfg.model
B, S, H, nh = cfg.micro_batch, m.seq_len, m.d_model, m.n_head
bf = torch.bfloat16
g = torch.Generator(device="cuda").manual_seed(0)
qkv = (torch.randn(B * S, 3 * H, device="cuda", generator=g) * 0.5).to(bf)
o = torch.empty(B * S, H, device="cuda", dtype=bf)
lse = torch.empty(B, nh, S, device="cuda")
do = (torch.randn(B * S, H, device="cuda", generator=g) * 0.5).to(bf)
dqkv = torch.empty_like(qkv)
for _ in range(reps):
    bb.op_attention_fwd("bf16", B, S, H, nh, bool(m.causal), qkv.data_ptr(), o.data_ptr(),
                        lse.data_ptr())
    bb.op_attention_bwd("bf16", B, S, H, nh, bool(m.causal), qkv.data_ptr(), o.data_ptr(),
                        lse.data_ptr(), do.data_ptr(), dqkv.data_ptr())
torch.cuda.synchronize()
print("ok", B, S, H, nh)
