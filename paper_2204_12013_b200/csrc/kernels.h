// kernels.h — launchers of the sm_100a kernels (host-callable, no templates).
// `bf16` selects the activation/parameter storage type: true = __nv_bfloat16
// (bf16 mode), false = float (fp32 check mode). Accumulation is fp32 always.
#pragma once
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>

namespace bb {
namespace k {

enum Epi : int { EPI_STORE = 0, EPI_BIAS = 1, EPI_BIAS_RES = 2, EPI_BIAS_GELU = 3,
                 EPI_GELU_BWD = 4, EPI_ACC_F32 = 5, EPI_STORE_F32 = 6 };

// D[m][n] = sum_k A(m,k) B(n,k); A(m,k) = A[m*lda+k] (a_mn=0) or A[k*lda+m] (a_mn=1).
struct Gemm {
  int M, N, K;
  const void *A; int lda; bool a_mn;
  const void *B; int ldb; bool b_mn;
  int epi;
  void *C; int ldc;
  const void *bias;   // [N] storage type
  const void *res;    // [M][ldc] storage type (EPI_BIAS_RES)
  void *aux;          // pre-activation [M][ldc] storage type (BIAS_GELU out, GELU_BWD in)
  bool tile_grid = false;   // one CTA (pair) per output tile instead of a persistent grid:
                            // a low-priority stream's GEMM then yields SMs tile by tile
  unsigned *trace = nullptr;   // BB_GEMM_TRACE: per-CTA progress words (mapped host memory)
  bool m_fast = false;         // set by the launcher: tile order walks M fastest (see gemm_tc)
};

// BB_GEMM_TRACE diagnostics: print the GEMM launches that have not finished.
void gemm_trace_dump();

// Profile mode: park a stream for `ns` of device time (not counted as a launch).
cudaError_t gpu_sleep(unsigned long long ns, cudaStream_t s);

// Global launch counter (kernels launched by this library in this process).
extern long long g_launches;

cudaError_t gemm_simt(bool bf16, const Gemm &g, cudaStream_t s);
cudaError_t gemm_tc(const Gemm &g, cudaStream_t s);        // bf16, tcgen05 + TMA
bool gemm_tc_supported(const Gemm &g);

cudaError_t embed_fwd(bool bf16, int R, int S, int H, const int32_t *tok, const void *E,
                      const void *Pos, void *x, cudaStream_t s);
// Deterministic embedding backward: tokens of the micro-batch grouped by id
// through a device-built CSR blob per micro-batch (embed_csr_ints(R) ints:
// uniq[R] | offs[R+1] | pos[R] | U), positions ascending within a group.
size_t embed_csr_ints(int R);
cudaError_t embed_csr(int M, int R, const int32_t *tok, int32_t *blob, cudaStream_t s);
cudaError_t embed_bwd(bool bf16, bool dx_f32, int R, int S, int H, const int32_t *csr,
                      const void *dx, float *dE, float *dPos, cudaStream_t s);

cudaError_t layernorm_fwd(bool bf16, int R, int H, const void *x, const void *g, const void *b,
                          void *y, float *mean, float *rstd, cudaStream_t s);
// dx = dres + LN'(dy). dy is fp32 (a GEMM output); the residual gradient
// dres is fp32 (dres32) or storage type (dresT) or absent; dx is written in
// the storage type (dxT, a GEMM operand) and, if dx32 != null, in fp32 too
// (the residual-gradient chain stays fp32 inside a stage).
cudaError_t layernorm_bwd_dx(bool bf16, int R, int H, const float *dy, const void *x,
                             const float *mean, const float *rstd, const void *g,
                             const float *dres32, const void *dresT, void *dxT, float *dx32,
                             cudaStream_t s);
// Deterministic column reductions through `partial` (>= colreduce_partial_floats
// floats, ZERO-INITIALISED once at allocation: its tail holds self-resetting
// arrival counters):
//   mode 0: out[n] += sum_r A[r][n]                     (bias gradient)
//   mode 1: out[n] += sum_r A[r][n] * (X[r][n]-mean[r])*rstd[r]   (LN gamma gradient)
// One launch when N % 8 == 0: row-block partials, and the last row block to
// arrive at a column block adds the partials in ascending row-block order.
size_t colreduce_partial_floats(int R, int N);
// a_f32: A is fp32 (else storage type); X is always storage type.
cudaError_t colreduce(bool bf16, bool a_f32, int mode, int R, int N, const void *A, const void *X,
                      const float *mean, const float *rstd, float *partial, float *out,
                      cudaStream_t s);
// Both LN parameter gradients in one pass over fp32 dA: out_g (mode 1), out_b (mode 0).
cudaError_t colreduce_ln(bool bf16, int R, int N, const float *A, const void *X, const float *mean,
                         const float *rstd, float *partial, float *out_g, float *out_b,
                         cudaStream_t s);

cudaError_t attention_fwd(bool bf16, int B, int S, int H, int nh, bool causal, const void *qkv,
                          void *o, float *lse, cudaStream_t s);
// scratch: B*nh*S floats.
// Scratch floats attention_bwd needs (row dots D, and for the tcgen05 path an
// fp32 dQ accumulator and ordering counters).
size_t attention_bwd_scratch_floats(int B, int S, int H, int nh);
cudaError_t attention_bwd(bool bf16, int B, int S, int H, int nh, bool causal, const void *qkv,
                          const void *o, const float *lse, const void *dout, void *dqkv,
                          float *scratch, cudaStream_t s);

cudaError_t cross_entropy(bool bf16, int R, int V, void *logits, const int32_t *targets,
                          float inv_ntok, float *loss_rows, cudaStream_t s);
// out[0] = sum of x[0..n) in a fixed order (single block).
cudaError_t sum_fixed(int n, const float *x, float *out, cudaStream_t s);

// D > 1 pipelines: dst = ((src[0] + src[1]) + src[2]) + ... over the
// D contributions in ascending pipeline order, fp32 (every pipeline computes
// the same bits). D <= kMaxPipelines; dst may alias none of the sources.
constexpr int kMaxPipelines = 8;
cudaError_t sum_pipelines(size_t n, const float *const *src, int D, float *dst, cudaStream_t s);

cudaError_t adam(size_t n, float *p, const float *g, float *m, float *v, void *w16, float lr,
                 float b1, float b2, float eps, float bc1, float bc2, cudaStream_t s);
cudaError_t cast_f32_to_bf16(size_t n, const float *src, void *dst, cudaStream_t s);
cudaError_t fill_nan(void *p, size_t bytes, cudaStream_t s);

}  // namespace k
}  // namespace bb
