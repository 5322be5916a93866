"""Debug aid: attention fwd/bwd through the C ABI vs a torch fp32 autograd
reference; prints the error of dQ / dK / dV per 128-row block.

    python tools/attn_bwd_check.py [B S nh causal]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2204_12013_b200 as bb  # noqa: E402

a = [int(x) for x in sys.argv[1:]] or [1, 256, 1, 1]
B, S, nh, causal = a
d = 64
H = nh * d
torch.manual_seed(0)
qkv = (torch.randn(B * S, 3 * H, device="cuda") * 0.5).to(torch.bfloat16)
do = (torch.randn(B * S, H, device="cuda") * 0.5).to(torch.bfloat16)
o = torch.zeros(B * S, H, device="cuda", dtype=torch.bfloat16)
lse = torch.zeros(B, nh, S, device="cuda")
dqkv = torch.zeros_like(qkv)
bb.op_attention_fwd("bf16", B, S, H, nh, bool(causal), qkv.data_ptr(), o.data_ptr(), lse.data_ptr())
bb.op_attention_bwd("bf16", B, S, H, nh, bool(causal), qkv.data_ptr(), o.data_ptr(), lse.data_ptr(),
                    do.data_ptr(), dqkv.data_ptr())
torch.cuda.synchronize()

x = qkv.float().view(B, S, 3, nh, d).permute(2, 0, 3, 1, 4).contiguous().requires_grad_(True)
q, k, v = x[0], x[1], x[2]
s = q @ k.transpose(-1, -2) / d ** 0.5
if causal:
    s = s.masked_fill(torch.triu(torch.ones(S, S, device="cuda", dtype=torch.bool), 1), float("-inf"))
p = torch.softmax(s, -1)
out = p @ v
out.backward(do.float().view(B, S, nh, d).permute(0, 2, 1, 3))
g = x.grad.permute(1, 3, 0, 2, 4).reshape(B * S, 3 * H)
got = dqkv.float()
o_ref = out.permute(0, 2, 1, 3).reshape(B * S, H)
print("o   max err", (o.float() - o_ref).abs().max().item(), "ref max", o_ref.abs().max().item())
for name, c in (("dQ", 0), ("dK", 1), ("dV", 2)):
    ref = g[:, c * H:(c + 1) * H]
    e = (got[:, c * H:(c + 1) * H] - ref).abs()
    blocks = [round(e[i:i + 128].max().item(), 4) for i in range(0, B * S, 128)]
    print(f"{name} max err {e.max().item():.4f} (ref max {ref.abs().max().item():.3f}) per block {blocks}")

# ---- diagnostics for dQ (first 128 queries of sequence 0, head 0)
if os.environ.get("DQDIAG"):
    with torch.no_grad():
        qq, kk_, vv = q[0, 0].detach(), k[0, 0].detach(), v[0, 0].detach()
        dO = do.float().view(B, S, nh, d)[0, :, 0]
        P = p[0, 0].detach()
        dP = dO @ vv.T
        Dq = (dO * o_ref.view(B, S, nh, d)[0, :, 0]).sum(-1, keepdim=True)
        dS = P * (dP - Dq)
        ref = g[:128, :d]
        gq = got[:128, :d]
        print("check ref == dS K / 8:", (dS[:128] @ kk_ / 8 - ref).abs().max().item())
        cands = {
            "dS^T K": (dS[:128, :128].T @ kk_[:128]) / 8,
            "atoms swapped": (torch.cat([dS[:128, 64:128], dS[:128, :64]], 1) @ kk_[:128]) / 8,
            "q-half swapped rows": torch.cat([ref[64:], ref[:64]]),
            "zero": torch.zeros_like(ref),
        }
        for nm, c in cands.items():
            print(f"  {nm:22s} err {(gq - c).abs().max().item():.4f}")
        print("  got/ref norm", (gq.norm() / ref.norm()).item())
        print("  per 8-row group err", [round((gq - ref)[i:i + 8].abs().max().item(), 4) for i in range(0, 128, 8)])
        print("  per 8-col group err", [round((gq - ref)[:, i:i + 8].abs().max().item(), 4) for i in range(0, 64, 8)])
