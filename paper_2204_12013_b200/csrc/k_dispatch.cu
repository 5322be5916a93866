// k_dispatch.cu — picks the kernel implementation per op and shape.
#include "k_common.cuh"

namespace bb {
namespace k {

cudaError_t attention_simt_fwd(bool bf16, int B, int S, int H, int nh, bool causal,
                               const void *qkv, void *o, float *lse, cudaStream_t s);
cudaError_t attention_simt_bwd(bool bf16, int B, int S, int H, int nh, bool causal,
                               const void *qkv, const void *o, const float *lse,
                               const void *dout, void *dqkv, float *scratch, cudaStream_t s);

cudaError_t attention_fwd(bool bf16, int B, int S, int H, int nh, bool causal, const void *qkv,
                          void *o, float *lse, cudaStream_t s) {
  return attention_simt_fwd(bf16, B, S, H, nh, causal, qkv, o, lse, s);
}

cudaError_t attention_bwd(bool bf16, int B, int S, int H, int nh, bool causal, const void *qkv,
                          const void *o, const float *lse, const void *dout, void *dqkv,
                          float *scratch, cudaStream_t s) {
  return attention_simt_bwd(bf16, B, S, H, nh, causal, qkv, o, lse, dout, dqkv, scratch, s);
}

}  // namespace k
}  // namespace bb
