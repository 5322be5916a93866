// k_attn_bwd_umma.cu — flash attention backward on the 5th-generation tensor
// cores (tcgen05 / TMEM / TMA), head dim 64, bf16 in, fp32 accumulation,
// deterministic.
//
// One CTA = one key block of 128 keys of one (sequence, head); it walks the
// query blocks (128 queries) that see those keys. Per query block i:
//   S^T  = K Q_i^T     (M=128 keys, N=128 queries, K=64)   -> TMEM
//   dP^T = V dO_i^T    (same shape)                         -> TMEM
//   softmax warps: P^T = exp(S^T * scale - LSE_q) (bf16 into TMEM),
//                  dS^T = P^T (dP^T - D_q) (bf16 into a double-buffered
//                  128B-swizzled K-major smem tile)
//   dV  += P^T dO_i    (M=128 keys, N=64, K=128 queries; A from TMEM)
//   dK  += dS^T Q_i                                          TMEM accumulator
//   dQ_i = dS K        (M=128 queries, N=64, K=128 keys; A = dS^T tile read
//                       MN-major)                            -> TMEM
//   dQ warps: scale and write the fp32 partial to the workspace slot of
//   (query block i, key block kb); the last contributor reduces (below).
// Determinism: the key blocks contributing to query block i write their dQ_i
// partials into separate workspace slots; whichever contributor arrives last
// (atomic ticket per query block and row quarter) sums the slots in ascending
// key-block order and writes dQ_i in bf16. No CTA ever waits on another.
// dK, dV leave TMEM once, at the end.
//
// Warps: 0 TMA producer (Q, dO boxes; LSE / D rows by bulk copy, or plain
// loads with +inf / 0 padding for a ragged S), 1 MMA issuer (one lane),
// 2..9 softmax (warp w: key rows 32 (w % 4).., query half (w - 2) / 4),
// 10..13 dQ epilogue (query rows 32 (w % 4)..).
// D_q = sum_d dO_q,d O_q,d comes from fa_bwd_d_kernel (k_attn_tc.cu).
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "k_common.cuh"
#include "k_sm100.cuh"

namespace bb {
namespace k {
cudaError_t attention_bwd_rowdot(int B, int S, int H, int nh, const void *o, const void *dout,
                                 float *Dv, cudaStream_t s);
namespace {
using namespace sm100;

constexpr int D = 64, BLK = 128, NST = 3;   // NST: Q / dO / LSE / D ring depth
constexpr int kThreads = 14 * 32;
constexpr float LOG2E = 1.4426950408889634f;

constexpr uint32_t idesc_f16(int m, int n, bool a_mn, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

struct Smem {
  static constexpr int K = 0;                          // 128 x 64 bf16, 16 KB
  static constexpr int V = K + 16384;
  static constexpr int Q = V + 16384;                  // NST stages x 16 KB
  static constexpr int DO = Q + NST * 16384;           // NST stages x 16 KB
  static constexpr int DST = DO + NST * 16384;         // 2 x dS^T 128 x 128 bf16 (2 atoms each)
  static constexpr int LSED = DST + 2 * 32768;         // NST stages x (128 LSE + 128 D) fp32
  static constexpr int BAR = LSED + NST * 2 * BLK * 4;
  static constexpr int BYTES = BAR + 256 + 1024;
};

// TMEM address of this warp's P^T columns: lanes of its quarter, 32 columns
// (64 queries as bf16 pairs) per query half g.
__device__ __forceinline__ uint32_t t_p_base(uint32_t t_pt, uint32_t lane_off, int g) {
  return t_pt + lane_off + 32 * g;
}

__device__ __forceinline__ uint32_t pack_bf2(float lo, float hi) {
  uint32_t r;   // one F2FP: hi -> upper half, lo -> lower half, round to nearest even
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
// 2^x, flush-to-zero approximation (MUFU.EX2 only): the arguments are
// s*scale - LSE <= ~0, far from the denormal range that matters here.
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 14 warps: at most 4 per SM sub-partition, so 128 registers per thread.
__global__ void __launch_bounds__(kThreads, 1)
    fa_bwd_umma_kernel(const __grid_constant__ CUtensorMap map_qkv,
                       const __grid_constant__ CUtensorMap map_do, float *__restrict__ ws,
                       int S, int H, int nh, int causal, int bulk_rows, int dbg,
                       const float *__restrict__ lse, const float *__restrict__ Dv,
                       __nv_bfloat16 *__restrict__ dqkv, unsigned long long *__restrict__ trace) {
  using L = Smem;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t *gbase = smem_raw + (base - raw);
  const uint32_t bars = base + L::BAR;
  const uint32_t kv_full = bars;
  auto qdo_full = [&](int s) { return bars + 8u * (1 + s); };
  auto qdo_empty = [&](int s) { return bars + 8u * (1 + NST + s); };
  const uint32_t sdp_full = bars + 8u * (1 + 2 * NST), pds_full = sdp_full + 8u,
                 dv_done = sdp_full + 16u, dq_full = sdp_full + 24u, dq_free = sdp_full + 32u,
                 fin = sdp_full + 40u;
  auto ds_free = [&](int b2) { return sdp_full + 48u + 8u * b2; };
  const uint32_t s_full = sdp_full, dp_full = sdp_full + 64u, s_free = sdp_full + 72u;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(gbase + L::BAR + 8 * (1 + 2 * NST + 10));
  float *lsed = reinterpret_cast<float *>(gbase + L::LSED);

  const int nkb = (S + BLK - 1) / BLK;
  // longest CTAs first (causal: key block 0 sees every query block): all
  // (sequence, head) pairs of key block 0, then of key block 1, ...
  const int kb = blockIdx.y, h = blockIdx.x % nh, b = blockIdx.x / nh;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int i0 = causal ? kb : 0;                 // first query block
  const int n = nkb - i0;                         // query blocks (steps)
  const size_t bh = (size_t)b * nh + h;
  const float scale = rsqrtf((float)D), sl2 = scale * LOG2E;

  if (warp == 0 && lane == 0) {
    mbar_init(kv_full, 1);
    for (int s = 0; s < NST; ++s) {
      mbar_init(qdo_full(s), 1);
      mbar_init(qdo_empty(s), 1);
    }
    mbar_init(s_full, 1);
    mbar_init(dp_full, 1);
    mbar_init(s_free, 8);
    mbar_init(pds_full, 8);
    mbar_init(dv_done, 1);
    mbar_init(ds_free(0), 1);
    mbar_init(ds_free(1), 1);
    mbar_init(dq_full, 1);
    mbar_init(dq_free, 4);
    mbar_init(fin, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_qkv)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_do)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  auto stamp = [&](int k) {            // BB_ATTN_DBG & 4: per-CTA timeline (64 slots)
    if (trace) {
      unsigned long long tt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
      trace[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 64 + k] = tt;
    }
  };
  // TMEM columns: S^T | dP^T (128 each) | dV | dK | dQ (64 each) | P^T (bf16 pairs, 64)
  const uint32_t t_s = tmem, t_dp = tmem + 128, t_dv = tmem + 256, t_dk = tmem + 320,
                 t_dq = tmem + 384, t_pt = tmem + 448;

  if (warp == 0) {
    // ---------------- producer: K, V once; then Q_i, dO_i, LSE_i, D_i per step
    if (lane == 0) {
      mbar_expect_tx(kv_full, 2 * 16384);
      tma_load_3d(base + L::K, &map_qkv, kv_full, H + h * D, kb * BLK, b);
      tma_load_3d(base + L::V, &map_qkv, kv_full, 2 * H + h * D, kb * BLK, b);
    }
    for (int t = 0; t < n; ++t) {
      const int i = i0 + t, st = t % NST;
      mbar_wait(qdo_empty(st), ((t / NST) & 1) ^ 1);
      float *ls = lsed + st * 2 * BLK;
      const uint32_t lsa = base + L::LSED + st * 2 * BLK * 4;
      if (!bulk_rows) {
        // ragged S: rows past S get LSE = +inf (P = 0, dS = 0) and D = 0
#pragma unroll
        for (int c = 0; c < BLK / 32; ++c) {
          const int qi = c * 32 + lane, q = i * BLK + qi;
          ls[qi] = q < S ? lse[bh * S + q] : INFINITY;
          ls[BLK + qi] = q < S ? Dv[bh * S + q] : 0.f;
        }
        __syncwarp();
      }
      if (lane == 0) {
        mbar_expect_tx(qdo_full(st), 2 * 16384 + (bulk_rows ? 2 * BLK * 4 : 0));
        tma_load_3d(base + L::Q + st * 16384, &map_qkv, qdo_full(st), h * D, i * BLK, b);
        tma_load_3d(base + L::DO + st * 16384, &map_do, qdo_full(st), h * D, i * BLK, b);
        if (bulk_rows) {
          bulk_load(lsa, lse + bh * S + i * BLK, BLK * 4, qdo_full(st));
          bulk_load(lsa + BLK * 4, Dv + bh * S + i * BLK, BLK * 4, qdo_full(st));
        }
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (lane == 0) {
      const uint32_t id_s = idesc_f16(128, BLK, false, false);
      const uint32_t id_kv = idesc_f16(128, D, false, true);    // dV, dK: B = dO / Q MN-major
      const uint32_t id_q = idesc_f16(128, D, true, true);      // dQ: A = dS (from dS^T), B = K
      // S^T(t+1) is issued as soon as the softmax warps hold S^T(t) in
      // registers (s_free), dP^T(t+1) once they are done with step t.
      auto issue_s = [&](int t) {
        const int st = t % NST;
        mbar_wait(qdo_full(st), (t / NST) & 1);
        tc_fence_after();
        const uint32_t q = base + L::Q + st * 16384;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_bf16(t_s, smem_desc(base + L::K + kk * 32, 16, 1024), smem_desc(q + kk * 32, 16, 1024),
                   id_s, kk > 0 ? 1u : 0u);
        mma_commit(s_full);
      };
      auto issue_dp = [&](int t) {      // Q/dO stage t already waited by issue_s(t)
        const uint32_t d = base + L::DO + (t % NST) * 16384;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_bf16(t_dp, smem_desc(base + L::V + kk * 32, 16, 1024),
                   smem_desc(d + kk * 32, 16, 1024), id_s, kk > 0 ? 1u : 0u);
        mma_commit(dp_full);
      };
      stamp(0);
      mbar_wait(kv_full, 0);
      stamp(1);
      issue_s(0);
      issue_dp(0);
      for (int t = 0; t < n; ++t) {
        const int st = t % NST;
        if (t + 1 < n) {
          mbar_wait_spin(s_free, t & 1);  // S^T(t) is in the softmax warps' registers
          tc_fence_after();
          issue_s(t + 1);
        }
        mbar_wait_spin(pds_full, t & 1);  // P^T, dS^T written; dP^T read out
        if (t < 8) stamp(2 + t);
        tc_fence_after();
        if (t + 1 < n) issue_dp(t + 1);
        const uint32_t q = base + L::Q + st * 16384, d = base + L::DO + st * 16384;
        const uint32_t dst = base + L::DST + (t & 1) * 32768;
        // dV += P^T dO_i: A = P^T from TMEM (16 queries = 8 columns per K step)
#pragma unroll
        for (int kk = 0; kk < BLK / 16; ++kk)
          mma_bf16_ts(t_dv, t_pt + kk * 8, smem_desc(d + kk * 2048, 8192, 1024), id_kv,
                      (t > 0 || kk > 0) ? 1u : 0u);
        mma_commit(dv_done);
        if (t > 0) {
          mbar_wait_spin(dq_free, (t - 1) & 1);
          tc_fence_after();
        }
        if (t < 8) stamp(10 + t);
#pragma unroll
        for (int kk = 0; kk < BLK / 16; ++kk) {
          // A = dS (queries x keys) read MN-major from the dS^T tile: 64-query
          // chunks 16 KB apart (LBO), 16 keys = 16 rows of 128 B per K step.
          const uint64_t a = smem_desc(dst + kk * 2048, 16384, 1024);
          const uint64_t bk = smem_desc(base + L::K + kk * 2048, 8192, 1024);
          mma_bf16(t_dq, a, bk, id_q, kk > 0 ? 1u : 0u);
        }
        mma_commit(dq_full);
#pragma unroll
        for (int kk = 0; kk < BLK / 16; ++kk) {
          // A: K-major 128 x 128 dS^T tile = two 64-query swizzle atoms 16 KB apart
          const uint32_t aoff = (kk / 4) * 16384 + (kk % 4) * 32;
          mma_bf16(t_dk, smem_desc(dst + aoff, 16, 1024), smem_desc(q + kk * 2048, 8192, 1024),
                   id_kv, (t > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(ds_free(t & 1));
        mma_commit(qdo_empty(st));
      }
      mma_commit(fin);
      if (trace) {
        uint32_t sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        stamp(60);
        trace[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 64 + 61] = sm;
      }
    }
  } else if (warp < 10) {
    // ---------------- softmax warps
    const int quarter = warp % 4, g = (warp - 2) / 4;
    const int r = quarter * 32 + lane;               // key row
    const int key = kb * BLK + r;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    for (int t = 0; t < n; ++t) {
      const int i = i0 + t, st = t % NST;
      const bool diag = causal && i == kb;
      const float *ls = lsed + st * 2 * BLK;
      mbar_wait(s_full, t & 1);
      const bool tr = warp == 2 && lane == 0 && t < 8;
      if (tr) stamp(20 + t);
      tc_fence_after();
      // (a) S^T row of this warp's 64 queries, one TMEM round trip, then
      // release S^T so the MMA warp can compute S^T(t+1) meanwhile
      float p[64];
      {
        uint32_t sv[4][16];
#pragma unroll
        for (int hh = 0; hh < 4; ++hh) tmem_ld16_nowait(t_s + lane_off + 64 * g + 16 * hh, sv[hh]);
        tmem_wait_ld();
#pragma unroll
        for (int hh = 0; hh < 4; ++hh) tmem_pin16(sv[hh]);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(s_free);
#pragma unroll
        for (int c = 0; c < 64; c += 4) {
          const float4 a = *reinterpret_cast<const float4 *>(ls + 64 * g + c);
          const float l2[4] = {a.x * LOG2E, a.y * LOG2E, a.z * LOG2E, a.w * LOG2E};
#pragma unroll
          for (int j = 0; j < 4; ++j)
            p[c + j] = ex2(fmaf(__uint_as_float(sv[(c + j) / 16][(c + j) % 16]), sl2, -l2[j]));
        }
      }
      if (diag) {                                     // causal diagonal block: key > query -> 0
#pragma unroll
        for (int c = 0; c < 64; ++c)
          if (key > i * BLK + 64 * g + c) p[c] = 0.f;
      }
      // P^T -> TMEM once dV of the previous step has read it
      if (t > 0) mbar_wait(dv_done, (t - 1) & 1);
      tc_fence_after();
      if (tr) stamp(28 + t);
#pragma unroll
      for (int hh = 0; hh < 4; ++hh) {
        uint32_t pp[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) pp[c] = pack_bf2(p[16 * hh + 2 * c], p[16 * hh + 2 * c + 1]);
        tmem_st8_nowait(t_p_base(t_pt, lane_off, g) + 8 * hh, pp);
      }
      // (b) dS^T = P^T (dP^T - D) -> smem buffer t & 1 (free once dQ / dK of
      // step t - 2 have read it); dP^T chunks pipelined against the math
      mbar_wait(dp_full, t & 1);
      if (t > 1) mbar_wait(ds_free(t & 1), ((t >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t drow = base + L::DST + (t & 1) * 32768 + g * 16384 + r * 128;
      uint32_t dv[2][16];
      tmem_ld16_nowait(t_dp + lane_off + 64 * g, dv[0]);
      tmem_wait_ld();
      tmem_pin16(dv[0]);
#pragma unroll
      for (int hh = 0; hh < 4; ++hh) {
        const int cur = hh & 1;
        if (hh < 3) tmem_ld16_nowait(t_dp + lane_off + 64 * g + 16 * (hh + 1), dv[cur ^ 1]);
        uint32_t dd[8];
#pragma unroll
        for (int c = 0; c < 16; c += 2) {
          const int qc = 64 * g + 16 * hh + c;
          dd[c / 2] = pack_bf2(p[16 * hh + c] * (__uint_as_float(dv[cur][c]) - ls[BLK + qc]),
                               p[16 * hh + c + 1] * (__uint_as_float(dv[cur][c + 1]) - ls[BLK + qc + 1]));
        }
        st_shared_v4(drow + (uint32_t)(((2 * hh) ^ (r & 7)) * 16), dd[0], dd[1], dd[2], dd[3]);
        st_shared_v4(drow + (uint32_t)(((2 * hh + 1) ^ (r & 7)) * 16), dd[4], dd[5], dd[6], dd[7]);
        if (hh < 3) {
          tmem_wait_ld();
          tmem_pin16(dv[cur ^ 1]);
        }
      }
      fence_async_smem();
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (tr) stamp(36 + t);
      if (lane == 0) mbar_arrive(pds_full);
    }
    // ---------------- dV (group 0) / dK (group 1) out of TMEM, once
    mbar_wait(fin, 0);
    tc_fence_after();
    const uint32_t src = g == 0 ? t_dv : t_dk;
    const float f = g == 0 ? 1.f : scale;
    __nv_bfloat16 *dst = dqkv + ((size_t)b * S + key) * 3 * H + (g == 0 ? 2 * H : H) + h * D;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      uint32_t v[32];
      tmem_ld32_nowait(src + lane_off + 32 * half, v);
      tmem_wait_ld();
      tmem_pin(v);
      if (key < S) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          *reinterpret_cast<uint4 *>(dst + 32 * half + 8 * c) = make_uint4(
              pack_bf2(__uint_as_float(v[8 * c]) * f, __uint_as_float(v[8 * c + 1]) * f),
              pack_bf2(__uint_as_float(v[8 * c + 2]) * f, __uint_as_float(v[8 * c + 3]) * f),
              pack_bf2(__uint_as_float(v[8 * c + 4]) * f, __uint_as_float(v[8 * c + 5]) * f),
              pack_bf2(__uint_as_float(v[8 * c + 6]) * f, __uint_as_float(v[8 * c + 7]) * f));
      }
    }
  } else {
    // ---------------- dQ epilogue: query row 32 quarter + lane of block i.
    // Every contributing key block writes its (scaled) dQ_i partial into its
    // own slot of a workspace; the last of the contributors' warps for this
    // (query block, row quarter) to arrive (atomic ticket) adds the slots in
    // ascending key-block order and writes bf16 dQ rows: no cross-CTA waits,
    // deterministic whatever the arrival order.
    const int quarter = warp % 4;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    for (int t = 0; t < n; ++t) {
      const int i = i0 + t;
      float *slot0 = ws + ((bh * nkb + i) * nkb) * (size_t)(BLK * D) + (size_t)(quarter * 32 + lane) * D;
      mbar_wait(dq_full, t & 1);
      tc_fence_after();
      uint32_t v[64];
      tmem_ld32_nowait(t_dq + lane_off, *reinterpret_cast<uint32_t(*)[32]>(v));
      tmem_ld32_nowait(t_dq + lane_off + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
      tmem_wait_ld();
      tmem_pin(*reinterpret_cast<uint32_t(*)[32]>(v));
      tmem_pin(*reinterpret_cast<uint32_t(*)[32]>(v + 32));
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dq_free);
      if (dbg & 1) continue;
      float4 *mine = reinterpret_cast<float4 *>(slot0 + (size_t)kb * BLK * D);
#pragma unroll
      for (int c = 0; c < D / 4; ++c)
        __stcg(mine + c, make_float4(__uint_as_float(v[4 * c]) * scale,
                                     __uint_as_float(v[4 * c + 1]) * scale,
                                     __uint_as_float(v[4 * c + 2]) * scale,
                                     __uint_as_float(v[4 * c + 3]) * scale));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// dQ rows: sum the contributing key blocks' fp32 partials in ascending
// key-block order, write bf16 into the Q block of dqkv. One thread = 8
// columns of one query row.
__global__ void dq_reduce_kernel(int B, int S, int H, int nh, int causal,
                                 const float *__restrict__ ws, __nv_bfloat16 *__restrict__ dqkv) {
  const int nkb = (S + BLK - 1) / BLK;
  const size_t total = (size_t)B * S * nh * (D / 8);
  for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < total;
       v += (size_t)gridDim.x * blockDim.x) {
    const int c8 = v % (D / 8);
    const size_t r = v / (D / 8);                 // (b, s, h) with h fastest
    const int h = r % nh;
    const size_t bs = r / nh;
    const int s = bs % S, b = bs / S;
    const int i = s / BLK, qr = s % BLK;
    const int nc = causal ? i + 1 : nkb;
    const size_t bh = (size_t)b * nh + h;
    const float *src = ws + ((bh * nkb + i) * nkb) * (size_t)(BLK * D) + (size_t)qr * D + 8 * c8;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int k2 = 0; k2 < nc; ++k2) {
      const float4 x = __ldcs(reinterpret_cast<const float4 *>(src + (size_t)k2 * BLK * D));
      const float4 y = __ldcs(reinterpret_cast<const float4 *>(src + (size_t)k2 * BLK * D + 4));
      acc[0] += x.x; acc[1] += x.y; acc[2] += x.z; acc[3] += x.w;
      acc[4] += y.x; acc[5] += y.y; acc[6] += y.z; acc[7] += y.w;
    }
    *reinterpret_cast<uint4 *>(dqkv + bs * 3 * H + h * D + 8 * c8) =
        make_uint4(pack_bf2(acc[0], acc[1]), pack_bf2(acc[2], acc[3]), pack_bf2(acc[4], acc[5]),
                   pack_bf2(acc[6], acc[7]));
  }
}
}  // namespace

bool attention_umma_bwd_supported(int B, int S, int H, int nh) {
  return H / nh == D && H % 8 == 0 && S >= 1 && B >= 1;
}

// Scratch (floats): D [B nh S] | dQ partial slots [B nh nkb nkb 128 64]
// (slot kb of query block i holds key block kb's dQ_i partial).
static int dbg_flags() {
  static const int f = [] {
    const char *e = std::getenv("BB_ATTN_DBG");
    return e ? std::atoi(e) : 0;
  }();
  return f;
}

// BB_ATTN_DBG & 4: per-CTA globaltimer stamps (start, K/V in, each step's
// softmax hand-off, end, SM id), written to bwd_trace.bin after each call.
static unsigned long long *g_trace = nullptr;
static size_t g_trace_n = 0;
static unsigned long long *trace_buf(size_t ctas) {
  if (!(dbg_flags() & 4)) return nullptr;
  if (g_trace_n < ctas) {
    if (g_trace) cudaFree(g_trace);
    cudaMalloc(&g_trace, ctas * 64 * 8);
    g_trace_n = ctas;
  }
  cudaMemset(g_trace, 0, ctas * 64 * 8);
  return g_trace;
}

size_t attention_umma_bwd_scratch_floats(int B, int S, int H, int nh) {
  const size_t nkb = (S + BLK - 1) / BLK;
  auto up = [](size_t x) { return (x + 63) / 64 * 64; };
  (void)H;
  return up((size_t)B * nh * S) + (size_t)B * nh * nkb * nkb * BLK * D;
}

cudaError_t attention_umma_bwd(int B, int S, int H, int nh, bool causal, const void *qkv,
                               const void *o, const float *lse, const void *dout, void *dqkv,
                               float *scratch, cudaStream_t s) {
  const int nkb = (S + BLK - 1) / BLK;
  auto up = [](size_t x) { return (x + 63) / 64 * 64; };
  float *Dv = scratch;
  float *ws = scratch + up((size_t)B * nh * S);
  CUtensorMap mq, md;
  {
    const uint64_t dims[3] = {(uint64_t)3 * H, (uint64_t)S, (uint64_t)B};
    const uint64_t st[2] = {(uint64_t)3 * H * 2, (uint64_t)S * 3 * H * 2};
    const uint32_t box[3] = {64, BLK, 1};
    if (!tma_map_3d(&mq, qkv, false, dims, st, box)) {
      fprintf(stderr, "[bb] attention bwd: qkv tensor map rejected\n");
      return cudaErrorInvalidValue;
    }
  }
  {
    const uint64_t dims[3] = {(uint64_t)H, (uint64_t)S, (uint64_t)B};
    const uint64_t st[2] = {(uint64_t)H * 2, (uint64_t)S * H * 2};
    const uint32_t box[3] = {64, BLK, 1};
    if (!tma_map_3d(&md, dout, false, dims, st, box)) {
      fprintf(stderr, "[bb] attention bwd: dO tensor map rejected\n");
      return cudaErrorInvalidValue;
    }
  }
  cudaError_t e = attention_bwd_rowdot(B, S, H, nh, o, dout, Dv, s);
  if (e != cudaSuccess) return e;
  static bool attr = false;
  if (!attr) {
    e = cudaFuncSetAttribute(fa_bwd_umma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             Smem::BYTES);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid(nh * B, nkb);
  fa_bwd_umma_kernel<<<grid, kThreads, Smem::BYTES, s>>>(
      mq, md, ws, S, H, nh, causal ? 1 : 0,
      (S % BLK == 0 && (reinterpret_cast<uintptr_t>(lse) & 15) == 0 &&
       (reinterpret_cast<uintptr_t>(Dv) & 15) == 0) ? 1 : 0,
      dbg_flags(), lse, Dv,
      reinterpret_cast<__nv_bfloat16 *>(dqkv), trace_buf(grid.x * grid.y));
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "[bb] attention bwd launch: %s\n", cudaGetErrorString(e));
    return e;
  }
  if (dbg_flags() & 4) {
    cudaStreamSynchronize(s);
    std::vector<unsigned long long> h((size_t)grid.x * grid.y * 64);
    cudaMemcpy(h.data(), g_trace, h.size() * 8, cudaMemcpyDeviceToHost);
    if (FILE *f = fopen("bwd_trace.bin", "wb")) {
      const int dims[4] = {(int)grid.x, (int)grid.y, nh, B};
      fwrite(dims, sizeof(int), 4, f);
      fwrite(h.data(), 8, h.size(), f);
      fclose(f);
    }
  }
  const size_t total = (size_t)B * S * nh * (D / 8);
  dq_reduce_kernel<<<(unsigned)std::min<size_t>((total + 255) / 256, 148 * 8), 256, 0, s>>>(
      B, S, H, nh, causal ? 1 : 0, ws, reinterpret_cast<__nv_bfloat16 *>(dqkv));
  g_launches += 2;
  return cudaGetLastError();
}

}  // namespace k
}  // namespace bb
