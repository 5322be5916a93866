// k_dispatch.cu — picks the kernel implementation per op and shape.
#include <algorithm>
#include <cstdlib>

#include "k_common.cuh"

namespace bb {
namespace k {

cudaError_t attention_simt_fwd(bool bf16, int B, int S, int H, int nh, bool causal,
                               const void *qkv, void *o, float *lse, cudaStream_t s);
cudaError_t attention_simt_bwd(bool bf16, int B, int S, int H, int nh, bool causal,
                               const void *qkv, const void *o, const float *lse,
                               const void *dout, void *dqkv, float *scratch, cudaStream_t s);

bool attention_tc_supported(int H, int nh);
cudaError_t attention_tc_fwd(int B, int S, int H, int nh, bool causal, const void *qkv, void *o,
                             float *lse, cudaStream_t s);
cudaError_t attention_tc_bwd(int B, int S, int H, int nh, bool causal, const void *qkv,
                             const void *o, const float *lse, const void *dout, void *dqkv,
                             float *scratch, cudaStream_t s);

bool attention_umma_supported(int B, int S, int H, int nh);
cudaError_t attention_umma_fwd(int B, int S, int H, int nh, bool causal, const void *qkv, void *o,
                               float *lse, cudaStream_t s);

bool attention_umma_bwd_supported(int B, int S, int H, int nh);
size_t attention_umma_bwd_scratch_floats(int B, int S, int H, int nh);
cudaError_t attention_umma_bwd(int B, int S, int H, int nh, bool causal, const void *qkv,
                               const void *o, const float *lse, const void *dout, void *dqkv,
                               float *scratch, cudaStream_t s);

size_t attention_bwd_scratch_floats(int B, int S, int H, int nh) {
  return std::max((size_t)B * nh * S, attention_umma_bwd_scratch_floats(B, S, H, nh));
}

// Explicit dispatch by head dimension, no silent fallbacks:
//  * bf16, head dim 64 (every GPT-2 / BERT config, C1-C3): tcgen05 kernels
//    (k_attn_umma.cu, k_attn_bwd_umma.cu); a token count below one 128-row
//    tile (B*S < 128, only in op-level tests) takes the mma.sync kernel;
//  * bf16, head dim 32 (only the tiny C0 model: 64 / 2 heads): mma.sync
//    tensor-core kernels (k_attn_tc.cu);
//  * fp32 check mode: exact-fp32 SIMT kernels by definition (Q9);
//  * anything else: cudaErrorNotSupported (bb_init rejects it up front).
cudaError_t attention_fwd(bool bf16, int B, int S, int H, int nh, bool causal, const void *qkv,
                          void *o, float *lse, cudaStream_t s) {
  if (!bf16) return attention_simt_fwd(false, B, S, H, nh, causal, qkv, o, lse, s);
  if (attention_umma_supported(B, S, H, nh))
    return attention_umma_fwd(B, S, H, nh, causal, qkv, o, lse, s);
  if (attention_tc_supported(H, nh))
    return attention_tc_fwd(B, S, H, nh, causal, qkv, o, lse, s);
  return cudaErrorNotSupported;
}

cudaError_t attention_bwd(bool bf16, int B, int S, int H, int nh, bool causal, const void *qkv,
                          const void *o, const float *lse, const void *dout, void *dqkv,
                          float *scratch, cudaStream_t s) {
  if (!bf16)
    return attention_simt_bwd(false, B, S, H, nh, causal, qkv, o, lse, dout, dqkv, scratch, s);
  if (attention_umma_bwd_supported(B, S, H, nh))
    return attention_umma_bwd(B, S, H, nh, causal, qkv, o, lse, dout, dqkv, scratch, s);
  if (attention_tc_supported(H, nh))
    return attention_tc_bwd(B, S, H, nh, causal, qkv, o, lse, dout, dqkv, scratch, s);
  return cudaErrorNotSupported;
}

}  // namespace k
}  // namespace bb
