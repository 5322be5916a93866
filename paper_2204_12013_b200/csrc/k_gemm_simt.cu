// k_gemm_simt.cu — fp32-FMA tiled GEMM for the fp32 check mode (SURVEY.md
// §2.2 K21: tcgen05 kind::tf32 has a 10-bit mantissa and cannot meet 1e-5),
// all operand layouts and epilogues. Deterministic: each output element sums
// k in ascending order in fp32.
#include "k_common.cuh"

namespace bb {
namespace k {

long long g_launches = 0;

namespace {
constexpr int BM = 64, BN = 64, BK = 16, TPB = 256;

template <typename T>
__global__ void __launch_bounds__(TPB) gemm_simt_kernel(Gemm g) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const T *A = reinterpret_cast<const T *>(g.A);
  const T *B = reinterpret_cast<const T *>(g.B);
  float acc[4][4] = {};
  for (int k0 = 0; k0 < g.K; k0 += BK) {
#pragma unroll
    for (int i = 0; i < (BM * BK) / TPB; ++i) {
      const int e = tid + i * TPB;
      int m, kk;
      if (g.a_mn) { kk = e / BM; m = e % BM; } else { m = e / BK; kk = e % BK; }
      const int gm = m0 + m, gk = k0 + kk;
      float v = 0.f;
      if (gm < g.M && gk < g.K)
        v = to_f(g.a_mn ? A[(size_t)gk * g.lda + gm] : A[(size_t)gm * g.lda + gk]);
      As[kk][m] = v;
    }
#pragma unroll
    for (int i = 0; i < (BN * BK) / TPB; ++i) {
      const int e = tid + i * TPB;
      int n, kk;
      if (g.b_mn) { kk = e / BN; n = e % BN; } else { n = e / BK; kk = e % BK; }
      const int gn = n0 + n, gk = k0 + kk;
      float v = 0.f;
      if (gn < g.N && gk < g.K)
        v = to_f(g.b_mn ? B[(size_t)gk * g.ldb + gn] : B[(size_t)gn * g.ldb + gk]);
      Bs[kk][n] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int m = m0 + ty + 16 * i, n = n0 + tx + 16 * j;
      if (m < g.M && n < g.N) epi_store<T>(g, m, n, acc[i][j]);
    }
}
}  // namespace

cudaError_t gemm_simt(bool bf16, const Gemm &g, cudaStream_t s) {
  if (g.M <= 0 || g.N <= 0) return cudaSuccess;
  dim3 grid((g.N + BN - 1) / BN, (g.M + BM - 1) / BM);
  if (bf16)
    gemm_simt_kernel<__nv_bfloat16><<<grid, TPB, 0, s>>>(g);
  else
    gemm_simt_kernel<float><<<grid, TPB, 0, s>>>(g);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace k
}  // namespace bb
