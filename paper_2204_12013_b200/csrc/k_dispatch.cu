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

static bool use_umma() {
  static const bool on = [] {
    const char *e = std::getenv("BB_ATTN_UMMA");
    return !(e && e[0] == '0');
  }();
  return on;
}

size_t attention_bwd_scratch_floats(int B, int S, int H, int nh) {
  return std::max((size_t)B * nh * S, attention_umma_bwd_scratch_floats(B, S, H, nh));
}

// bf16: tcgen05 flash attention forward (head dim 64), else the mma.sync
// kernels (head dim 32/64); fp32 check mode: SIMT.
cudaError_t attention_fwd(bool bf16, int B, int S, int H, int nh, bool causal, const void *qkv,
                          void *o, float *lse, cudaStream_t s) {
  // tcgen05 kernels (k_attn_umma.cu, k_attn_bwd_umma.cu) for head dim 64;
  // BB_ATTN_UMMA=0 selects the mma.sync kernels instead (tests / comparisons).
  if (bf16 && use_umma() && attention_umma_supported(B, S, H, nh))
    return attention_umma_fwd(B, S, H, nh, causal, qkv, o, lse, s);
  if (bf16 && attention_tc_supported(H, nh))
    return attention_tc_fwd(B, S, H, nh, causal, qkv, o, lse, s);
  return attention_simt_fwd(bf16, B, S, H, nh, causal, qkv, o, lse, s);
}

cudaError_t attention_bwd(bool bf16, int B, int S, int H, int nh, bool causal, const void *qkv,
                          const void *o, const float *lse, const void *dout, void *dqkv,
                          float *scratch, cudaStream_t s) {
  if (bf16 && use_umma() && attention_umma_bwd_supported(B, S, H, nh))
    return attention_umma_bwd(B, S, H, nh, causal, qkv, o, lse, dout, dqkv, scratch, s);
  if (bf16 && attention_tc_supported(H, nh))
    return attention_tc_bwd(B, S, H, nh, causal, qkv, o, lse, dout, dqkv, scratch, s);
  return attention_simt_bwd(bf16, B, S, H, nh, causal, qkv, o, lse, dout, dqkv, scratch, s);
}

}  // namespace k
}  // namespace bb
