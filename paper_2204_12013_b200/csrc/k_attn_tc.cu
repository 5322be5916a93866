// k_attn_tc.cu — bf16 flash attention forward / backward on tensor cores
// (warp-level mma.sync m16n8k16, fp32 accumulation), head dim 32 or 64.
//
// Forward: one CTA = 64 query rows of one (sequence, head), 4 warps x 16 rows;
// loop over 64-key blocks with an online softmax (P kept in registers as the
// A operand of P.V), O and the log-sum-exp written at the end.
// Backward, deterministic (no atomics): D_i = do_i.o_i;
// kernel dQ: one CTA per 64 query rows loops over key blocks; kernel dK/dV:
// one CTA per 64 keys loops over query blocks. P is recomputed from the LSE.
#include "k_common.cuh"

namespace bb {
namespace k {
namespace {

constexpr int BQ = 64, BKV = 64, NT = 128;
constexpr float LOG2E = 1.4426950408889634f;

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t *>(&v);
}

__device__ __forceinline__ uint32_t ld32(const __nv_bfloat16 *p) {
  return *reinterpret_cast<const uint32_t *>(p);
}

// A-operand fragments of a 16 x D row block (rows r0.., columns = head dims)
// read straight from global memory (rows >= S give zeros).
template <int D>
__device__ __forceinline__ void load_rows_frag(uint32_t (&f)[D / 16][4],
                                               const __nv_bfloat16 *base, size_t ld, int r0,
                                               int S, int g, int t) {
#pragma unroll
  for (int ks = 0; ks < D / 16; ++ks) {
    const int c = ks * 16 + 2 * t;
    const bool ok0 = r0 + g < S, ok1 = r0 + g + 8 < S;
    f[ks][0] = ok0 ? ld32(base + (size_t)(r0 + g) * ld + c) : 0u;
    f[ks][1] = ok1 ? ld32(base + (size_t)(r0 + g + 8) * ld + c) : 0u;
    f[ks][2] = ok0 ? ld32(base + (size_t)(r0 + g) * ld + c + 8) : 0u;
    f[ks][3] = ok1 ? ld32(base + (size_t)(r0 + g + 8) * ld + c + 8) : 0u;
  }
}

// Copy a 64 x D tile (rows r0.., stride ld) into row-major smem [64][D+8]
// and/or transposed smem [D][64+8]. Rows >= S are zero.
template <int D>
__device__ __forceinline__ void load_tile(__nv_bfloat16 (*rowm)[D + 8],
                                          __nv_bfloat16 (*trans)[BKV + 8],
                                          const __nv_bfloat16 *base, size_t ld, int r0, int S) {
  constexpr int V8 = D / 8;
  for (int i = threadIdx.x; i < 64 * V8; i += NT) {
    const int r = i / V8, c8 = (i % V8) * 8;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r0 + r < S) v = *reinterpret_cast<const uint4 *>(base + (size_t)(r0 + r) * ld + c8);
    if (rowm) *reinterpret_cast<uint4 *>(&rowm[r][c8]) = v;
    if (trans) {
      const __nv_bfloat16 *e = reinterpret_cast<const __nv_bfloat16 *>(&v);
#pragma unroll
      for (int j = 0; j < 8; ++j) trans[c8 + j][r] = e[j];
    }
  }
}

// ------------------------------------------------------------------ forward
template <int D>
__global__ void __launch_bounds__(NT) fa_fwd_kernel(int S, int H, int nh, int causal,
                                                    const __nv_bfloat16 *__restrict__ qkv,
                                                    __nv_bfloat16 *__restrict__ o,
                                                    float *__restrict__ lse) {
  __shared__ __align__(16) __nv_bfloat16 Ks[BKV][D + 8];
  __shared__ __align__(16) __nv_bfloat16 Vt[D][BKV + 8];
  const int qb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, g = lane >> 2, t = lane & 3;
  const size_t ld = 3 * (size_t)H;
  const __nv_bfloat16 *Q = qkv + (size_t)b * S * ld + h * D;
  const __nv_bfloat16 *K = Q + H, *V = Q + 2 * H;
  const int q0 = qb * BQ + warp * 16;
  uint32_t qf[D / 16][4];
  load_rows_frag<D>(qf, Q, ld, q0, S, g, t);
  const float sl2 = rsqrtf((float)D) * LOG2E;
  float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
  float acc[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
  const int nkb_all = (S + BKV - 1) / BKV;
  const int nkb = causal ? min(nkb_all, qb + 1) : nkb_all;
  for (int kb = 0; kb < nkb; ++kb) {
    __syncthreads();
    load_tile<D>(Ks, nullptr, K, ld, kb * BKV, S);
    load_tile<D>(nullptr, Vt, V, ld, kb * BKV, S);
    __syncthreads();
    float s[8][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks)
        mma16816(s[nt], qf[ks], ld32(&Ks[nt * 8 + g][ks * 16 + 2 * t]),
                 ld32(&Ks[nt * 8 + g][ks * 16 + 8 + 2 * t]));
    }
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = kb * BKV + nt * 8 + 2 * t + (e & 1);
        const int row = q0 + g + (e >> 1) * 8;
        float v = s[nt][e] * sl2;
        if (key >= S || (causal && key > row)) v = -INFINITY;
        s[nt][e] = v;
        mx[e >> 1] = fmaxf(mx[e >> 1], v);
      }
    float corr[2], mnew[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
      mnew[r] = fmaxf(m[r], mx[r]);
      corr[r] = mnew[r] == -INFINITY ? 1.f : exp2f(m[r] - mnew[r]);
      m[r] = mnew[r];
      l[r] *= corr[r];
    }
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      acc[i][0] *= corr[0];
      acc[i][1] *= corr[0];
      acc[i][2] *= corr[1];
      acc[i][3] *= corr[1];
    }
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float mr = m[e >> 1];
        const float p = mr == -INFINITY ? 0.f : exp2f(s[nt][e] - mr);
        s[nt][e] = p;
        l[e >> 1] += p;
      }
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t a[4] = {pack_bf16(s[2 * kk][0], s[2 * kk][1]), pack_bf16(s[2 * kk][2], s[2 * kk][3]),
                       pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]),
                       pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3])};
#pragma unroll
      for (int dn = 0; dn < D / 8; ++dn)
        mma16816(acc[dn], a, ld32(&Vt[dn * 8 + g][kk * 16 + 2 * t]),
                 ld32(&Vt[dn * 8 + g][kk * 16 + 8 + 2 * t]));
    }
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l[r] += __shfl_xor_sync(0xffffffffu, l[r], 1);
    l[r] += __shfl_xor_sync(0xffffffffu, l[r], 2);
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int row = q0 + g + r * 8;
    if (row >= S) continue;
    const float inv = 1.f / l[r];
    __nv_bfloat16 *orow = o + ((size_t)b * S + row) * H + h * D;
#pragma unroll
    for (int dn = 0; dn < D / 8; ++dn)
      *reinterpret_cast<uint32_t *>(orow + dn * 8 + 2 * t) =
          pack_bf16(acc[dn][2 * r] * inv, acc[dn][2 * r + 1] * inv);
    if (t == 0) lse[((size_t)b * nh + h) * S + row] = (m[r] + log2f(l[r])) / LOG2E;
  }
}

// D_i = sum_d do[i,d] * o[i,d]; one warp per row.
__global__ void fa_bwd_d_kernel(int R, int S, int H, int nh, const __nv_bfloat16 *__restrict__ o,
                                const __nv_bfloat16 *__restrict__ dout, float *__restrict__ Dv) {
  const int row = blockIdx.x * 4 + threadIdx.x / 32;   // over B*S*nh
  const int lane = threadIdx.x % 32;
  if (row >= R * nh) return;
  const int h = row % nh, r = row / nh;   // r = b*S + i
  const int d = H / nh;
  const size_t off = (size_t)r * H + h * d;
  float s = 0.f;
  for (int c = lane; c < d; c += 32) s += __bfloat162float(o[off + c]) * __bfloat162float(dout[off + c]);
  s = warp_sum(s);
  const int b = r / S, i = r % S;
  if (lane == 0) Dv[((size_t)b * nh + h) * S + i] = s;
}

// ------------------------------------------------------------ backward: dQ
template <int D>
__global__ void __launch_bounds__(NT) fa_bwd_dq_kernel(int S, int H, int nh, int causal,
                                                       const __nv_bfloat16 *__restrict__ qkv,
                                                       const __nv_bfloat16 *__restrict__ dout,
                                                       const float *__restrict__ lse,
                                                       const float *__restrict__ Dv,
                                                       __nv_bfloat16 *__restrict__ dqkv) {
  __shared__ __align__(16) __nv_bfloat16 Ks[BKV][D + 8];
  __shared__ __align__(16) __nv_bfloat16 Kt[D][BKV + 8];
  __shared__ __align__(16) __nv_bfloat16 Vs[BKV][D + 8];
  const int qb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, g = lane >> 2, t = lane & 3;
  const size_t ld = 3 * (size_t)H;
  const __nv_bfloat16 *Q = qkv + (size_t)b * S * ld + h * D;
  const __nv_bfloat16 *K = Q + H, *V = Q + 2 * H;
  const __nv_bfloat16 *dO = dout + (size_t)b * S * H + h * D;
  const int q0 = qb * BQ + warp * 16;
  uint32_t qf[D / 16][4], df[D / 16][4];
  load_rows_frag<D>(qf, Q, ld, q0, S, g, t);
  load_rows_frag<D>(df, dO, H, q0, S, g, t);
  const float scale = rsqrtf((float)D), sl2 = scale * LOG2E;
  float lrow[2], drow[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int row = q0 + g + r * 8;
    const size_t ri = ((size_t)b * nh + h) * S + min(row, S - 1);
    lrow[r] = lse[ri] * LOG2E;
    drow[r] = Dv[ri];
  }
  float acc[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
  const int nkb_all = (S + BKV - 1) / BKV;
  const int nkb = causal ? min(nkb_all, qb + 1) : nkb_all;
  for (int kb = 0; kb < nkb; ++kb) {
    __syncthreads();
    load_tile<D>(Ks, Kt, K, ld, kb * BKV, S);
    load_tile<D>(Vs, nullptr, V, ld, kb * BKV, S);
    __syncthreads();
    float s[8][4], dp[8][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) s[nt][e] = dp[nt][e] = 0.f;
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks) {
        mma16816(s[nt], qf[ks], ld32(&Ks[nt * 8 + g][ks * 16 + 2 * t]),
                 ld32(&Ks[nt * 8 + g][ks * 16 + 8 + 2 * t]));
        mma16816(dp[nt], df[ks], ld32(&Vs[nt * 8 + g][ks * 16 + 2 * t]),
                 ld32(&Vs[nt * 8 + g][ks * 16 + 8 + 2 * t]));
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = kb * BKV + nt * 8 + 2 * t + (e & 1);
        const int row = q0 + g + (e >> 1) * 8;
        float p = exp2f(s[nt][e] * sl2 - lrow[e >> 1]);
        if (key >= S || row >= S || (causal && key > row)) p = 0.f;
        s[nt][e] = p * (dp[nt][e] - drow[e >> 1]);   // dS
      }
    }
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t a[4] = {pack_bf16(s[2 * kk][0], s[2 * kk][1]), pack_bf16(s[2 * kk][2], s[2 * kk][3]),
                       pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]),
                       pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3])};
#pragma unroll
      for (int dn = 0; dn < D / 8; ++dn)
        mma16816(acc[dn], a, ld32(&Kt[dn * 8 + g][kk * 16 + 2 * t]),
                 ld32(&Kt[dn * 8 + g][kk * 16 + 8 + 2 * t]));
    }
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int row = q0 + g + r * 8;
    if (row >= S) continue;
    __nv_bfloat16 *dq = dqkv + ((size_t)b * S + row) * ld + h * D;
#pragma unroll
    for (int dn = 0; dn < D / 8; ++dn)
      *reinterpret_cast<uint32_t *>(dq + dn * 8 + 2 * t) =
          pack_bf16(acc[dn][2 * r] * scale, acc[dn][2 * r + 1] * scale);
  }
}

// --------------------------------------------------------- backward: dK, dV
template <int D>
__global__ void __launch_bounds__(NT) fa_bwd_dkv_kernel(int S, int H, int nh, int causal,
                                                        const __nv_bfloat16 *__restrict__ qkv,
                                                        const __nv_bfloat16 *__restrict__ dout,
                                                        const float *__restrict__ lse,
                                                        const float *__restrict__ Dv,
                                                        __nv_bfloat16 *__restrict__ dqkv) {
  __shared__ __align__(16) __nv_bfloat16 Qs[BQ][D + 8];
  __shared__ __align__(16) __nv_bfloat16 Qt[D][BQ + 8];
  __shared__ __align__(16) __nv_bfloat16 Ds[BQ][D + 8];
  __shared__ __align__(16) __nv_bfloat16 Dt[D][BQ + 8];
  __shared__ float ls[BQ], dsv[BQ];
  const int kb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, g = lane >> 2, t = lane & 3;
  const size_t ld = 3 * (size_t)H;
  const __nv_bfloat16 *Q = qkv + (size_t)b * S * ld + h * D;
  const __nv_bfloat16 *K = Q + H, *V = Q + 2 * H;
  const __nv_bfloat16 *dO = dout + (size_t)b * S * H + h * D;
  const int k0 = kb * BKV + warp * 16;
  uint32_t kf[D / 16][4], vf[D / 16][4];
  load_rows_frag<D>(kf, K, ld, k0, S, g, t);
  load_rows_frag<D>(vf, V, ld, k0, S, g, t);
  const float scale = rsqrtf((float)D), sl2 = scale * LOG2E;
  float dk[D / 8][4], dv[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.f;
  const int nqb = (S + BQ - 1) / BQ;
  for (int qb = causal ? kb : 0; qb < nqb; ++qb) {
    __syncthreads();
    load_tile<D>(Qs, Qt, Q, ld, qb * BQ, S);
    load_tile<D>(Ds, Dt, dO, H, qb * BQ, S);
    for (int i = threadIdx.x; i < BQ; i += NT) {
      const int q = qb * BQ + i;
      const size_t ri = ((size_t)b * nh + h) * S + min(q, S - 1);
      ls[i] = lse[ri] * LOG2E;
      dsv[i] = Dv[ri];
    }
    __syncthreads();
    float p[8][4], dp[8][4];   // transposed: rows = this warp's keys, cols = queries
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) p[nt][e] = dp[nt][e] = 0.f;
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks) {
        mma16816(p[nt], kf[ks], ld32(&Qs[nt * 8 + g][ks * 16 + 2 * t]),
                 ld32(&Qs[nt * 8 + g][ks * 16 + 8 + 2 * t]));
        mma16816(dp[nt], vf[ks], ld32(&Ds[nt * 8 + g][ks * 16 + 2 * t]),
                 ld32(&Ds[nt * 8 + g][ks * 16 + 8 + 2 * t]));
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int qi = nt * 8 + 2 * t + (e & 1);
        const int q = qb * BQ + qi;
        const int key = k0 + g + (e >> 1) * 8;
        float pv = exp2f(p[nt][e] * sl2 - ls[qi]);
        if (q >= S || key >= S || (causal && key > q)) pv = 0.f;
        p[nt][e] = pv;
        dp[nt][e] = pv * (dp[nt][e] - dsv[qi]);   // dS^T
      }
    }
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t ap[4] = {pack_bf16(p[2 * kk][0], p[2 * kk][1]), pack_bf16(p[2 * kk][2], p[2 * kk][3]),
                        pack_bf16(p[2 * kk + 1][0], p[2 * kk + 1][1]),
                        pack_bf16(p[2 * kk + 1][2], p[2 * kk + 1][3])};
      uint32_t as[4] = {pack_bf16(dp[2 * kk][0], dp[2 * kk][1]),
                        pack_bf16(dp[2 * kk][2], dp[2 * kk][3]),
                        pack_bf16(dp[2 * kk + 1][0], dp[2 * kk + 1][1]),
                        pack_bf16(dp[2 * kk + 1][2], dp[2 * kk + 1][3])};
#pragma unroll
      for (int dn = 0; dn < D / 8; ++dn) {
        mma16816(dv[dn], ap, ld32(&Dt[dn * 8 + g][kk * 16 + 2 * t]),
                 ld32(&Dt[dn * 8 + g][kk * 16 + 8 + 2 * t]));
        mma16816(dk[dn], as, ld32(&Qt[dn * 8 + g][kk * 16 + 2 * t]),
                 ld32(&Qt[dn * 8 + g][kk * 16 + 8 + 2 * t]));
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int key = k0 + g + r * 8;
    if (key >= S) continue;
    __nv_bfloat16 *dkr = dqkv + ((size_t)b * S + key) * ld + H + h * D;
    __nv_bfloat16 *dvr = dkr + H;
#pragma unroll
    for (int dn = 0; dn < D / 8; ++dn) {
      *reinterpret_cast<uint32_t *>(dkr + dn * 8 + 2 * t) =
          pack_bf16(dk[dn][2 * r] * scale, dk[dn][2 * r + 1] * scale);
      *reinterpret_cast<uint32_t *>(dvr + dn * 8 + 2 * t) =
          pack_bf16(dv[dn][2 * r], dv[dn][2 * r + 1]);
    }
  }
}

template <int D>
cudaError_t fwd_d(int B, int S, int H, int nh, bool causal, const void *qkv, void *o, float *lse,
                  cudaStream_t s) {
  dim3 grid((S + BQ - 1) / BQ, nh, B);
  fa_fwd_kernel<D><<<grid, NT, 0, s>>>(S, H, nh, causal, (const __nv_bfloat16 *)qkv,
                                       (__nv_bfloat16 *)o, lse);
  ++g_launches;
  return cudaGetLastError();
}

template <int D>
cudaError_t bwd_d(int B, int S, int H, int nh, bool causal, const void *qkv, const void *o,
                  const float *lse, const void *dout, void *dqkv, float *scratch, cudaStream_t s) {
  const int rows = B * S * nh;
  fa_bwd_d_kernel<<<(rows + 3) / 4, 128, 0, s>>>(B * S, S, H, nh, (const __nv_bfloat16 *)o,
                                                 (const __nv_bfloat16 *)dout, scratch);
  dim3 grid((S + BQ - 1) / BQ, nh, B);
  fa_bwd_dq_kernel<D><<<grid, NT, 0, s>>>(S, H, nh, causal, (const __nv_bfloat16 *)qkv,
                                          (const __nv_bfloat16 *)dout, lse, scratch,
                                          (__nv_bfloat16 *)dqkv);
  fa_bwd_dkv_kernel<D><<<grid, NT, 0, s>>>(S, H, nh, causal, (const __nv_bfloat16 *)qkv,
                                           (const __nv_bfloat16 *)dout, lse, scratch,
                                           (__nv_bfloat16 *)dqkv);
  g_launches += 3;
  return cudaGetLastError();
}
}  // namespace

bool attention_tc_supported(int H, int nh) {
  const int d = H / nh;
  return (d == 64 || d == 32) && H % 8 == 0;
}

cudaError_t attention_tc_fwd(int B, int S, int H, int nh, bool causal, const void *qkv, void *o,
                             float *lse, cudaStream_t s) {
  if (H / nh == 64) return fwd_d<64>(B, S, H, nh, causal, qkv, o, lse, s);
  return fwd_d<32>(B, S, H, nh, causal, qkv, o, lse, s);
}

cudaError_t attention_tc_bwd(int B, int S, int H, int nh, bool causal, const void *qkv,
                             const void *o, const float *lse, const void *dout, void *dqkv,
                             float *scratch, cudaStream_t s) {
  if (H / nh == 64) return bwd_d<64>(B, S, H, nh, causal, qkv, o, lse, dout, dqkv, scratch, s);
  return bwd_d<32>(B, S, H, nh, causal, qkv, o, lse, dout, dqkv, scratch, s);
}

}  // namespace k
}  // namespace bb
