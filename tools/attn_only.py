import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2204_12013_b200 as bb
B, S, H, nh = 8, 1024, 768, 12
bf = torch.bfloat16
qkv = (torch.randn(B * S, 3 * H, device="cuda") * 0.5).to(bf)
o = torch.empty(B * S, H, device="cuda", dtype=bf); lse = torch.empty(B, nh, S, device="cuda")
do = (torch.randn(B * S, H, device="cuda") * 0.5).to(bf); dqkv = torch.empty_like(qkv)
for _ in range(2):
    bb.op_attention_fwd("bf16", B, S, H, nh, True, qkv.data_ptr(), o.data_ptr(), lse.data_ptr())
    bb.op_attention_bwd("bf16", B, S, H, nh, True, qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), do.data_ptr(), dqkv.data_ptr())
torch.cuda.synchronize()
print("ok")
