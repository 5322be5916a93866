// k_attn_tc.cu — bf16 flash attention forward / backward on tensor cores
// (warp-level mma.sync m16n8k16, fp32 accumulation), head dim 32 or 64.
//
// Tiles of 64 keys (or queries) are copied row-major into padded shared
// memory with cp.async (double-buffered: the next tile streams in while the
// current one is consumed); MMA operands are read with ldmatrix (.trans where
// the operand is needed key-major), so no explicit transposes are stored.
// Forward: one CTA = 128 query rows (8 warps x 16) of one (sequence, head),
// online softmax in registers, P reused in registers as the A operand of P.V.
// Backward, deterministic (no atomics): D_i = do_i.o_i;
// dQ pass: CTA per 128 query rows loops over key tiles; dK/dV pass: CTA per
// 128 keys loops over query tiles. P is recomputed from the saved LSE.
#include "k_common.cuh"

namespace bb {
namespace k {
namespace {

constexpr int BR = 128;          // rows (queries or keys) per CTA, 16 per warp
constexpr int BT = 64;           // streamed tile (keys or queries)
constexpr int NW = BR / 16, NT = NW * 32;
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

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void *p) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void *p) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
}

__device__ __forceinline__ void cp_async16(void *dst, const void *src, bool ok) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src),
               "r"(ok ? 16 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N> __device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N));
}

template <int D> struct Tile { __nv_bfloat16 v[BT][D + 8]; };   // 16B-row padding: no ldsm conflicts

// Async copy of a 64 x D row tile (rows r0.., stride ld elements) into smem;
// rows >= S are zero-filled.
template <int D>
__device__ __forceinline__ void tile_async(Tile<D> &t, const __nv_bfloat16 *base, size_t ld,
                                           int r0, int S) {
  constexpr int V8 = D / 8;
  for (int i = threadIdx.x; i < BT * V8; i += NT) {
    const int r = i / V8, c8 = (i % V8) * 8;
    const bool ok = r0 + r < S;
    cp_async16(&t.v[r][c8], base + (size_t)(ok ? r0 + r : 0) * ld + c8, ok);
  }
}

// A-operand fragments of a warp's 16 x D row block read from global memory.
template <int D>
__device__ __forceinline__ void rows_frag(uint32_t (&f)[D / 16][4], const __nv_bfloat16 *base,
                                          size_t ld, int r0, int S, int g, int t) {
#pragma unroll
  for (int ks = 0; ks < D / 16; ++ks) {
    const int c = ks * 16 + 2 * t;
    const bool ok0 = r0 + g < S, ok1 = r0 + g + 8 < S;
    const __nv_bfloat16 *p0 = base + (size_t)(r0 + g) * ld + c;
    const __nv_bfloat16 *p1 = base + (size_t)(r0 + g + 8) * ld + c;
    f[ks][0] = ok0 ? *reinterpret_cast<const uint32_t *>(p0) : 0u;
    f[ks][1] = ok1 ? *reinterpret_cast<const uint32_t *>(p1) : 0u;
    f[ks][2] = ok0 ? *reinterpret_cast<const uint32_t *>(p0 + 8) : 0u;
    f[ks][3] = ok1 ? *reinterpret_cast<const uint32_t *>(p1 + 8) : 0u;
  }
}

// acc[16 x 8*NG] += A[16 x D] . T^T where T is a (8*NG) x D row tile starting at
// row r0 of `t` (B = T rows as columns: "S = Q K^T"). A given as D/16
// fragments. K-step outer, column groups inner: consecutive MMAs feed
// independent accumulators, and each K step's B fragments are loaded first.
template <int D, int NG = 8>
__device__ __forceinline__ void mma_abt(float (&acc)[NG][4], const uint32_t (&a)[D / 16][4],
                                        const Tile<D> &t, int lane, int r0 = 0) {
#pragma unroll
  for (int ks = 0; ks < D / 16; ++ks) {
    uint32_t r[NG / 2][4];
#pragma unroll
    for (int np = 0; np < NG / 2; ++np) {
      const int row = r0 + np * 16 + (lane & 7) + ((lane >> 4) << 3);
      const int col = ks * 16 + ((lane >> 3) & 1) * 8;
      ldsm_x4(r[np], &t.v[row][col]);
    }
#pragma unroll
    for (int np = 0; np < NG / 2; ++np) {
      mma16816(acc[2 * np], a[ks], r[np][0], r[np][1]);
      mma16816(acc[2 * np + 1], a[ks], r[np][2], r[np][3]);
    }
  }
}

// acc[16 x D] += P[16 x 16*KK] . T where T is a (16*KK) x D row tile starting
// at row r0 of `t`; P given as the fp32 accumulator layout of a 16 x (16*KK)
// block (converted to bf16 A fragments).
template <int D, int KK = 4>
__device__ __forceinline__ void mma_pt(float (&acc)[D / 8][4], const float (&p)[2 * KK][4],
                                       const Tile<D> &t, int lane, int r0 = 0) {
#pragma unroll
  for (int kk = 0; kk < KK; ++kk) {
    const uint32_t a[4] = {pack_bf16(p[2 * kk][0], p[2 * kk][1]),
                           pack_bf16(p[2 * kk][2], p[2 * kk][3]),
                           pack_bf16(p[2 * kk + 1][0], p[2 * kk + 1][1]),
                           pack_bf16(p[2 * kk + 1][2], p[2 * kk + 1][3])};
    uint32_t r[D / 16][4];
#pragma unroll
    for (int dp = 0; dp < D / 16; ++dp) {
      const int row = r0 + kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
      const int col = dp * 16 + (lane >> 4) * 8;
      ldsm_x4_t(r[dp], &t.v[row][col]);
    }
#pragma unroll
    for (int dp = 0; dp < D / 16; ++dp) {
      mma16816(acc[2 * dp], a, r[dp][0], r[dp][1]);
      mma16816(acc[2 * dp + 1], a, r[dp][2], r[dp][3]);
    }
  }
}

// ------------------------------------------------------------------ forward
template <int D>
__global__ void __launch_bounds__(NT, 2) fa_fwd_kernel(int S, int H, int nh, int causal,
                                                    const __nv_bfloat16 *__restrict__ qkv,
                                                    __nv_bfloat16 *__restrict__ o,
                                                    float *__restrict__ lse) {
  __shared__ __align__(128) Tile<D> Ks[2], Vs[2];
  const int qb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, g = lane >> 2, t = lane & 3;
  const size_t ld = 3 * (size_t)H;
  const __nv_bfloat16 *Q = qkv + (size_t)b * S * ld + h * D;
  const __nv_bfloat16 *K = Q + H, *V = Q + 2 * H;
  const int q0 = qb * BR + warp * 16;
  const int nkb_all = (S + BT - 1) / BT;
  const int nkb = causal ? min(nkb_all, ((qb + 1) * BR + BT - 1) / BT) : nkb_all;
  tile_async<D>(Ks[0], K, ld, 0, S);
  tile_async<D>(Vs[0], V, ld, 0, S);
  cp_commit();
  uint32_t qf[D / 16][4];
  rows_frag<D>(qf, Q, ld, q0, S, g, t);
  const float sl2 = rsqrtf((float)D) * LOG2E;
  float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
  float acc[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
  for (int kb = 0; kb < nkb; ++kb) {
    const int cur = kb & 1;
    if (kb + 1 < nkb) {
      tile_async<D>(Ks[cur ^ 1], K, ld, (kb + 1) * BT, S);
      tile_async<D>(Vs[cur ^ 1], V, ld, (kb + 1) * BT, S);
    }
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    const bool skip = causal && kb * BT > q0 + 15;   // whole tile above this warp's diagonal
    if (!skip) {
      float s[8][4];
#pragma unroll
      for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
      mma_abt<D>(s, qf, Ks[cur], lane);
      // scores stay unscaled; masks only on the diagonal / tail tiles
      if (kb * BT + BT > S || (causal && kb * BT + BT - 1 > q0)) {
#pragma unroll
        for (int nt = 0; nt < 8; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int key = kb * BT + nt * 8 + 2 * t + (e & 1);
            const int row = q0 + g + (e >> 1) * 8;
            if (key >= S || (causal && key > row)) s[nt][e] = -INFINITY;
          }
      }
      float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) mx[e >> 1] = fmaxf(mx[e >> 1], s[nt][e]);
      float corr[2], ms[2];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
        mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
        const float mn = fmaxf(m[r], mx[r]);
        corr[r] = mn == -INFINITY ? 1.f : exp2f((m[r] - mn) * sl2);
        ms[r] = mn == -INFINITY ? 0.f : mn * sl2;
        m[r] = mn;
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
          const float p = exp2f(fmaf(s[nt][e], sl2, -ms[e >> 1]));   // -inf -> 0
          s[nt][e] = p;
          l[e >> 1] += p;
        }
      mma_pt<D>(acc, s, Vs[cur], lane);
    }
    __syncthreads();
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
    if (t == 0) lse[((size_t)b * nh + h) * S + row] = (m[r] * sl2 + log2f(l[r])) / LOG2E;
  }
}

// D_i = sum_d do[i,d] * o[i,d]; one warp per (row, head).
__global__ void fa_bwd_d_kernel(int R, int S, int H, int nh, const __nv_bfloat16 *__restrict__ o,
                                const __nv_bfloat16 *__restrict__ dout, float *__restrict__ Dv) {
  const int row = blockIdx.x * 4 + threadIdx.x / 32;   // over B*S*nh
  const int lane = threadIdx.x % 32;
  if (row >= R * nh) return;
  const int h = row % nh, r = row / nh;   // r = b*S + i
  const int d = H / nh;
  const size_t off = (size_t)r * H + h * d;
  float s = 0.f;
  for (int c = 2 * lane; c < d; c += 64) {
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(o + off + c));
    const float2 x = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(dout + off + c));
    s += a.x * x.x + a.y * x.y;
  }
  s = warp_sum(s);
  const int b = r / S, i = r % S;
  if (lane == 0) Dv[((size_t)b * nh + h) * S + i] = s;
}

// ------------------------------------------------------------ backward: dQ
template <int D>
__global__ void __launch_bounds__(NT, 2) fa_bwd_dq_kernel(int S, int H, int nh, int causal,
                                                       const __nv_bfloat16 *__restrict__ qkv,
                                                       const __nv_bfloat16 *__restrict__ dout,
                                                       const float *__restrict__ lse,
                                                       const float *__restrict__ Dv,
                                                       __nv_bfloat16 *__restrict__ dqkv) {
  __shared__ __align__(128) Tile<D> Ks[2], Vs[2];
  const int qb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, g = lane >> 2, t = lane & 3;
  const size_t ld = 3 * (size_t)H;
  const __nv_bfloat16 *Q = qkv + (size_t)b * S * ld + h * D;
  const __nv_bfloat16 *K = Q + H, *V = Q + 2 * H;
  const __nv_bfloat16 *dO = dout + (size_t)b * S * H + h * D;
  const int q0 = qb * BR + warp * 16;
  const int nkb_all = (S + BT - 1) / BT;
  const int nkb = causal ? min(nkb_all, ((qb + 1) * BR + BT - 1) / BT) : nkb_all;
  tile_async<D>(Ks[0], K, ld, 0, S);
  tile_async<D>(Vs[0], V, ld, 0, S);
  cp_commit();
  uint32_t qf[D / 16][4], df[D / 16][4];
  rows_frag<D>(qf, Q, ld, q0, S, g, t);
  rows_frag<D>(df, dO, H, q0, S, g, t);
  const float scale = rsqrtf((float)D), sl2 = scale * LOG2E;
  float lrow[2], drow[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int row = min(q0 + g + r * 8, S - 1);
    const size_t ri = ((size_t)b * nh + h) * S + row;
    lrow[r] = lse[ri] * LOG2E;
    drow[r] = Dv[ri];
  }
  float acc[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
  for (int kb = 0; kb < nkb; ++kb) {
    const int cur = kb & 1;
    if (kb + 1 < nkb) {
      tile_async<D>(Ks[cur ^ 1], K, ld, (kb + 1) * BT, S);
      tile_async<D>(Vs[cur ^ 1], V, ld, (kb + 1) * BT, S);
    }
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    const bool skip = causal && kb * BT > q0 + 15;
    if (!skip) {
      float s[8][4], dp[8][4];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) s[i][e] = dp[i][e] = 0.f;
      mma_abt<D>(s, qf, Ks[cur], lane);
      mma_abt<D>(dp, df, Vs[cur], lane);
      const bool mask = kb * BT + BT > S || q0 + 16 > S || (causal && kb * BT + BT - 1 > q0);
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float p = exp2f(fmaf(s[nt][e], sl2, -lrow[e >> 1]));
          if (mask) {
            const int key = kb * BT + nt * 8 + 2 * t + (e & 1);
            const int row = q0 + g + (e >> 1) * 8;
            if (key >= S || row >= S || (causal && key > row)) p = 0.f;
          }
          s[nt][e] = p * (dp[nt][e] - drow[e >> 1]);   // dS
        }
      mma_pt<D>(acc, s, Ks[cur], lane);                // dQ += dS . K
    }
    __syncthreads();
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
__global__ void __launch_bounds__(NT, 2) fa_bwd_dkv_kernel(int S, int H, int nh, int causal,
                                                        const __nv_bfloat16 *__restrict__ qkv,
                                                        const __nv_bfloat16 *__restrict__ dout,
                                                        const float *__restrict__ lse,
                                                        const float *__restrict__ Dv,
                                                        __nv_bfloat16 *__restrict__ dqkv) {
  __shared__ __align__(128) Tile<D> Qs[2], Os[2];
  __shared__ float ls[2][BT], dsv[2][BT];
  const int kb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, g = lane >> 2, t = lane & 3;
  const size_t ld = 3 * (size_t)H;
  const __nv_bfloat16 *Q = qkv + (size_t)b * S * ld + h * D;
  const __nv_bfloat16 *K = Q + H, *V = Q + 2 * H;
  const __nv_bfloat16 *dO = dout + (size_t)b * S * H + h * D;
  const int k0 = kb * BR + warp * 16;
  const int nqb = (S + BT - 1) / BT;
  const int qb0 = causal ? (kb * BR) / BT : 0;
  auto stage = [&](int buf, int qb) {
    tile_async<D>(Qs[buf], Q, ld, qb * BT, S);
    tile_async<D>(Os[buf], dO, H, qb * BT, S);
    for (int i = threadIdx.x; i < BT; i += NT) {
      const int q = min(qb * BT + i, S - 1);
      const size_t ri = ((size_t)b * nh + h) * S + q;
      ls[buf][i] = lse[ri] * LOG2E;
      dsv[buf][i] = Dv[ri];
    }
  };
  if (qb0 < nqb) stage(0, qb0);
  cp_commit();
  uint32_t kf[D / 16][4], vf[D / 16][4];
  rows_frag<D>(kf, K, ld, k0, S, g, t);
  rows_frag<D>(vf, V, ld, k0, S, g, t);
  const float scale = rsqrtf((float)D), sl2 = scale * LOG2E;
  float dk[D / 8][4], dv[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.f;
  for (int qb = qb0; qb < nqb; ++qb) {
    const int cur = (qb - qb0) & 1;
    if (qb + 1 < nqb) stage(cur ^ 1, qb + 1);
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    const bool skip = causal && qb * BT + BT - 1 < k0;   // tile entirely before these keys
    if (!skip) {
#pragma unroll
      for (int hq = 0; hq < 2; ++hq) {     // two 32-query halves (register budget)
        if (causal && qb * BT + hq * 32 + 31 < k0) continue;
        float p[4][4], dp[4][4];   // transposed: rows = this warp's keys, cols = queries
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int e = 0; e < 4; ++e) p[i][e] = dp[i][e] = 0.f;
        mma_abt<D, 4>(p, kf, Qs[cur], lane, hq * 32);    // S^T = K Q^T
        mma_abt<D, 4>(dp, vf, Os[cur], lane, hq * 32);   // dP^T = V dO^T
        const int qlo = qb * BT + hq * 32;
        const bool mask = qlo + 32 > S || k0 + 16 > S || (causal && k0 + 15 > qlo);
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int qi = hq * 32 + nt * 8 + 2 * t + (e & 1);
            float pv = exp2f(fmaf(p[nt][e], sl2, -ls[cur][qi]));
            if (mask) {
              const int q = qb * BT + qi;
              const int key = k0 + g + (e >> 1) * 8;
              if (q >= S || key >= S || (causal && key > q)) pv = 0.f;
            }
            p[nt][e] = pv;
            dp[nt][e] = pv * (dp[nt][e] - dsv[cur][qi]);   // dS^T
          }
        mma_pt<D, 2>(dv, p, Os[cur], lane, hq * 32);    // dV += P^T dO
        mma_pt<D, 2>(dk, dp, Qs[cur], lane, hq * 32);   // dK += dS^T Q
      }
    }
    __syncthreads();
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
  dim3 grid((S + BR - 1) / BR, nh, B);
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
  dim3 grid((S + BR - 1) / BR, nh, B);
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

// D for head dim 64, 16-byte loads: 8 lanes per (row, head), 4 (row, head)
// pairs per warp; the 8 partial dots are added by a fixed xor tree.
__global__ void __launch_bounds__(256) fa_bwd_d64_kernel(int R, int S, int H, int nh,
                                                         const __nv_bfloat16 *__restrict__ o,
                                                         const __nv_bfloat16 *__restrict__ dout,
                                                         float *__restrict__ Dv) {
  const int gid = blockIdx.x * 32 + threadIdx.x / 8;   // (row, head) pair
  const int sub = threadIdx.x % 8;
  const bool ok = gid < R * nh;
  const int h = ok ? gid % nh : 0, r = ok ? gid / nh : 0;
  const size_t off = (size_t)r * H + h * 64 + sub * 8;
  float acc = 0.f;
  if (ok) {
    const uint4 a = *reinterpret_cast<const uint4 *>(o + off);
    const uint4 x = *reinterpret_cast<const uint4 *>(dout + off);
    const __nv_bfloat162 *pa = reinterpret_cast<const __nv_bfloat162 *>(&a);
    const __nv_bfloat162 *px = reinterpret_cast<const __nv_bfloat162 *>(&x);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 fa = __bfloat1622float2(pa[j]), fx = __bfloat1622float2(px[j]);
      acc += fa.x * fx.x + fa.y * fx.y;
    }
  }
#pragma unroll
  for (int m = 1; m < 8; m <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
  if (ok && sub == 0) {
    const int b = r / S, i = r % S;
    Dv[((size_t)b * nh + h) * S + i] = acc;
  }
}

cudaError_t attention_bwd_rowdot(int B, int S, int H, int nh, const void *o, const void *dout,
                                 float *Dv, cudaStream_t s) {
  const int rows = B * S * nh;
  if (H / nh == 64 && H % 8 == 0)
    fa_bwd_d64_kernel<<<(rows + 31) / 32, 256, 0, s>>>(B * S, S, H, nh, (const __nv_bfloat16 *)o,
                                                       (const __nv_bfloat16 *)dout, Dv);
  else
    fa_bwd_d_kernel<<<(rows + 3) / 4, 128, 0, s>>>(B * S, S, H, nh, (const __nv_bfloat16 *)o,
                                                   (const __nv_bfloat16 *)dout, Dv);
  ++g_launches;
  return cudaGetLastError();
}

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
