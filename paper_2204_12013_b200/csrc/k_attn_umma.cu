// k_attn_umma.cu — flash attention forward on the 5th-generation tensor cores
// (tcgen05 / TMEM / TMA), head dim 64, bf16 in, fp32 accumulation.
//
// One CTA = 128 query rows of one (sequence, head); key blocks of 128; two
// CTAs per SM (256 TMEM columns = S | P | O, ~81 KB smem each), so one CTA's
// softmax overlaps the other's MMAs.
//   warp 0      TMA: the Q tile once, then K_j and V_j into a 2-stage ring
//               (128B-swizzled, straight out of the packed [B*S, 3H] qkv);
//   warp 1      one lane issues S_j = Q K_j^T (M=128, N=128, K=64) into TMEM
//               as soon as the softmax has read S_{j-1}, then
//               O += P_{j-1} V_{j-1} (M=128, N=64, K=128; A = P from TMEM,
//               V = MN-major smem B) once P_{j-1} is in TMEM;
//   warps 2..9  softmax, two warps per TMEM lane quarter, each owning half of
//               the 128 key columns of a row (row max and row sum combined
//               through shared memory); thread r = query row r: pass 1 reads
//               its S row (4 x 32 columns) for the row max, pass 2 re-reads
//               it, exponentiates (exp2 of pre-scaled scores), packs P to
//               bf16 registers and releases S; then, once PV_{j-1} is done,
//               writes P_j to TMEM and rescales its O row if the max moved.
//               At the end: O / l and the log-sum-exp.
// Same math and LSE convention as the mma.sync kernel (k_attn_tc.cu), which
// the backward pass uses.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "k_common.cuh"
#include "k_sm100.cuh"

namespace bb {
namespace k {
namespace {
using namespace sm100;

constexpr int D = 64, BQ = 128, BKV = 128, ST = 2;
constexpr int kThreads = 64 + 8 * 32;   // producer, MMA, 8 softmax warps (2 per TMEM lane quarter)
constexpr float LOG2E = 1.4426950408889634f;

__device__ __forceinline__ uint32_t pack_bf2(float lo, float hi) {
  uint32_t r;   // one F2FP: hi -> upper half, lo -> lower half, round to nearest even
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
// 2^x on MUFU.EX2 alone (flush-to-zero): arguments are s*scale - max <= 0.
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

constexpr uint32_t idesc_f16(int m, int n, bool a_mn, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

struct SmemLayout {
  static constexpr int Q = 0;                         // 128 x 64 bf16 = 16 KB
  static constexpr int K = Q + BQ * D * 2;            // ST x 16 KB
  static constexpr int V = K + ST * BKV * D * 2;      // ST x 16 KB
  static constexpr int XCH = V + ST * BKV * D * 2;    // row-max / row-sum exchange (3 KB)
  static constexpr int BAR = XCH + (2 * 2 * BQ + 2 * BQ) * 4;
  static constexpr int BYTES = BAR + 128 + 1024;
};

__global__ void __launch_bounds__(kThreads, 2)
    fa_fwd_umma_kernel(const __grid_constant__ CUtensorMap map_qkv, int S, int H, int nh,
                       int causal, __nv_bfloat16 *__restrict__ o, float *__restrict__ lse,
                       unsigned long long *__restrict__ trace) {
  auto stamp = [&](int k) {            // BB_ATTN_DBG & 8: per-CTA timeline (64 slots)
    if (trace && k < 64) {
      unsigned long long tt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
      trace[((size_t)(blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * 64 + k] = tt;
    }
  };
  using L = SmemLayout;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t *gbase = smem_raw + (base - raw);
  const uint32_t bars = base + L::BAR;
  const uint32_t q_full = bars;
  // separate K and V rings: K_j is released by S_j (early), V_j by PV_j (late),
  // so K_{j+1} streams in while the softmax of block j-1 still runs
  auto k_full = [&](int s) { return bars + 8u * (1 + s); };
  auto v_full = [&](int s) { return bars + 8u * (1 + ST + s); };
  auto k_empty = [&](int s) { return bars + 8u * (1 + 2 * ST + s); };
  auto v_empty = [&](int s) { return bars + 8u * (1 + 3 * ST + s); };
  const uint32_t s_full = bars + 8u * (1 + 4 * ST);
  const uint32_t s_free = bars + 8u * (2 + 4 * ST);
  const uint32_t p_full = bars + 8u * (3 + 4 * ST);
  const uint32_t o_done = bars + 8u * (4 + 4 * ST);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(gbase + L::BAR + 8 * (5 + 4 * ST));

  // heaviest (causal: last) query blocks first, across the whole grid: the
  // query block is the slowest grid dimension, so the block scheduler hands
  // out every (head, sequence) of the last query block before any lighter one
  // (longest-processing-time-first packing of the 2-per-SM slots)
  const int qb = gridDim.z - 1 - blockIdx.z, h = blockIdx.x, b = blockIdx.y;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int q0 = qb * BQ;
  const int row_base = b * S;            // first qkv row of this sequence
  const int nkb_all = (S + BKV - 1) / BKV;
  const int nkb = causal ? min(nkb_all, (q0 + BQ - 1) / BKV + 1) : nkb_all;

  if (warp == 0 && lane == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < ST; ++s) {
      mbar_init(k_full(s), 1);
      mbar_init(v_full(s), 1);
      mbar_init(k_empty(s), 1);
      mbar_init(v_empty(s), 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_free, 8);     // one arrive per softmax warp
    mbar_init(p_full, 8);
    mbar_init(o_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_qkv)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM columns: S (fp32, 128) | P (bf16 pairs, 64) | O (fp32, 64)
  const uint32_t t_s = tmem, t_p = tmem + 128, t_o = tmem + 192;

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(q_full, BQ * D * 2);
      tma_load_2d(base + L::Q, &map_qkv, q_full, h * D, row_base + q0);
      for (int j = 0; j < nkb; ++j) {
        const int s = j % ST;
        mbar_wait(k_empty(s), ((j / ST) & 1) ^ 1);
        mbar_expect_tx(k_full(s), BKV * D * 2);
        tma_load_2d(base + L::K + s * BKV * D * 2, &map_qkv, k_full(s), H + h * D,
                    row_base + j * BKV);
        mbar_wait(v_empty(s), ((j / ST) & 1) ^ 1);
        mbar_expect_tx(v_full(s), BKV * D * 2);
        tma_load_2d(base + L::V + s * BKV * D * 2, &map_qkv, v_full(s), 2 * H + h * D,
                    row_base + j * BKV);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t id_s = idesc_f16(128, BKV, false, false);
      const uint32_t id_o = idesc_f16(128, D, false, true);
      auto issue_pv = [&](int j) {       // O += P_j V_j
        const int s = j % ST;
        mbar_wait(v_full(s), (j / ST) & 1);
        mbar_wait_spin(p_full, j & 1);
        if (j < 16) stamp(18 + j);
        tc_fence_after();
        const uint32_t va = base + L::V + s * BKV * D * 2;
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk) {
          // P from TMEM (16 keys = 8 columns per K step); V: MN-major,
          // 16 keys = 16 rows of 128 B per K step.
          const uint64_t db = smem_desc(va + kk * 2048, 8192, 1024);
          mma_bf16_ts(t_o, t_p + kk * 8, db, id_o, (j > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(o_done);
        mma_commit(v_empty(s));
      };
      stamp(0);
      mbar_wait(q_full, 0);
      stamp(1);
      for (int j = 0; j < nkb; ++j) {
        const int s = j % ST;
        mbar_wait(k_full(s), (j / ST) & 1);
        if (j > 0) mbar_wait_spin(s_free, (j - 1) & 1);    // S_{j-1} read out of TMEM
        tc_fence_after();
        const uint32_t ka = base + L::K + s * BKV * D * 2;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_bf16(t_s, smem_desc(base + L::Q + kk * 32, 16, 1024),
                   smem_desc(ka + kk * 32, 16, 1024), id_s, kk > 0 ? 1u : 0u);
        mma_commit(s_full);
        if (j < 16) stamp(2 + j);
        mma_commit(k_empty(s));
        if (j > 0) issue_pv(j - 1);
      }
      issue_pv(nkb - 1);
    }
  } else {
    // ---------------- softmax warps: row r = query q0 + r (TMEM lane r); the
    // two warps of a lane quarter split the 128 key columns (hf = half) and
    // combine row max / row sum through shared memory (named barrier 1 + q)
    const int q = warp % 4, hf = (warp - 2) / 4;
    const int r = q * 32 + lane;
    const int qrow = q0 + r;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const float sl2 = rsqrtf((float)D) * LOG2E;
    float *xm = reinterpret_cast<float *>(gbase + L::XCH);          // [2 parity][2 half][BQ]
    float *xl = xm + 2 * 2 * BQ;                                     // [2 half][BQ]
    float m = -INFINITY, l = 0.f;                                    // l: this half's partial sum
    for (int j = 0; j < nkb; ++j) {
      mbar_wait(s_full, j & 1);
      if (warp == 2 && lane == 0 && j < 14) stamp(34 + j);
      tc_fence_after();
      const bool need_mask = (j * BKV + BKV > S) || (causal && j * BKV + BKV - 1 > q0);
      const int kmax = causal ? min(S - 1, qrow) : S - 1;   // last valid key of this row
      const int k0 = j * BKV + 64 * hf;                      // first key of this half
      uint32_t t[64];
      tmem_ld32_nowait(t_s + lane_off + 64 * hf, *reinterpret_cast<uint32_t(*)[32]>(t));
      tmem_ld32_nowait(t_s + lane_off + 64 * hf + 32, *reinterpret_cast<uint32_t(*)[32]>(t + 32));
      tmem_wait_ld();
      tmem_pin(*reinterpret_cast<uint32_t(*)[32]>(t));
      tmem_pin(*reinterpret_cast<uint32_t(*)[32]>(t + 32));
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(s_free);            // S may be overwritten by S_{j+1}
      if (need_mask) {
#pragma unroll
        for (int i = 0; i < 64; ++i)
          if (k0 + i > kmax) t[i] = __float_as_uint(-INFINITY);
      }
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < 64; ++i) mx = fmaxf(mx, __uint_as_float(t[i]));
      xm[((j & 1) * 2 + hf) * BQ + r] = mx;
      asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
      mx = fmaxf(xm[((j & 1) * 2 + 0) * BQ + r], xm[((j & 1) * 2 + 1) * BQ + r]);
      const float mn = fmaxf(m, mx * sl2);
      const float corr = mn == -INFINITY ? 1.f : exp2f(m - mn);
      m = mn;
      const float mnz = mn == -INFINITY ? 0.f : mn;   // fully masked row: exp2(-inf) = 0
      // P = exp2(s * sl2 - m), packed to bf16 pairs in place
      float sum = 0.f;
#pragma unroll
      for (int i = 0; i < 64; i += 2) {
        const float p0 = ex2(fmaf(__uint_as_float(t[i]), sl2, -mnz));
        const float p1 = ex2(fmaf(__uint_as_float(t[i + 1]), sl2, -mnz));
        sum += p0 + p1;
        t[i / 2] = pack_bf2(p0, p1);
      }
      l = l * corr + sum;
      if (j > 0) {
        mbar_wait(o_done, (j - 1) & 1);    // PV_{j-1} done: O stable, P columns free
        tc_fence_after();
      }
      // this half's P -> TMEM (lane r, 32 columns of bf16 pairs)
      tmem_st32_nowait(t_p + lane_off + 32 * hf, t);
      if (j > 0 && __any_sync(0xffffffffu, corr != 1.f)) {   // this half's 32 O columns
        uint32_t ov[32];
        tmem_ld32_nowait(t_o + lane_off + 32 * hf, ov);
        tmem_wait_ld();
        tmem_pin(ov);
#pragma unroll
        for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * corr);
        tmem_st32_nowait(t_o + lane_off + 32 * hf, ov);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (warp == 2 && lane == 0 && j < 14) stamp(48 + j);
      if (lane == 0) mbar_arrive(p_full);
    }
    xl[hf * BQ + r] = l;
    asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");
    const float lt = xl[r] + xl[BQ + r];              // fixed order: half 0 + half 1
    mbar_wait(o_done, (nkb - 1) & 1);
    tc_fence_after();
    float ov[32];
    tmem_ld32(t_o + lane_off + 32 * hf, ov);
    if (qrow < S) {
      const float inv = 1.f / lt;
      __nv_bfloat16 *orow = o + ((size_t)row_base + qrow) * H + h * D + 32 * hf;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        *reinterpret_cast<uint4 *>(orow + 8 * c) =
            make_uint4(pack_bf2(ov[8 * c] * inv, ov[8 * c + 1] * inv),
                       pack_bf2(ov[8 * c + 2] * inv, ov[8 * c + 3] * inv),
                       pack_bf2(ov[8 * c + 4] * inv, ov[8 * c + 5] * inv),
                       pack_bf2(ov[8 * c + 6] * inv, ov[8 * c + 7] * inv));
      if (hf == 0) lse[((size_t)b * nh + h) * S + qrow] = (m + log2f(lt)) / LOG2E;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
  }
}
}  // namespace

bool attention_umma_supported(int B, int S, int H, int nh) {
  return H / nh == D && H % 8 == 0 && S >= 1 && (long)B * S >= BQ;
}

cudaError_t attention_umma_fwd(int B, int S, int H, int nh, bool causal, const void *qkv, void *o,
                               float *lse, cudaStream_t s) {
  CUtensorMap map;
  if (!tma_map_bf16_2d(&map, qkv, (uint64_t)3 * H, (uint64_t)B * S, (uint64_t)3 * H, 128))
    return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(fa_fwd_umma_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         SmemLayout::BYTES);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid(nh, B, (S + BQ - 1) / BQ);
  static const bool tr = [] {
    const char *e = std::getenv("BB_ATTN_DBG");
    return e && (std::atoi(e) & 8);
  }();
  static unsigned long long *tbuf = nullptr;
  static size_t tn = 0;
  const size_t ctas = (size_t)grid.x * grid.y * grid.z;
  if (tr && tn < ctas) {
    if (tbuf) cudaFree(tbuf);
    cudaMalloc(&tbuf, ctas * 64 * 8);
    tn = ctas;
  }
  if (tr) cudaMemsetAsync(tbuf, 0, ctas * 64 * 8, s);
  fa_fwd_umma_kernel<<<grid, kThreads, SmemLayout::BYTES, s>>>(
      map, S, H, nh, causal ? 1 : 0, reinterpret_cast<__nv_bfloat16 *>(o), lse,
      tr ? tbuf : nullptr);
  ++g_launches;
  if (tr) {   // write fwd_trace.bin: dims, then 64 stamps per CTA
    cudaStreamSynchronize(s);
    std::vector<unsigned long long> h(ctas * 64);
    cudaMemcpy(h.data(), tbuf, h.size() * 8, cudaMemcpyDeviceToHost);
    if (FILE *f = fopen("fwd_trace.bin", "wb")) {
      const int dims[3] = {(int)grid.x, (int)grid.y, (int)grid.z};
      fwrite(dims, sizeof(int), 3, f);
      fwrite(h.data(), 8, h.size(), f);
      fclose(f);
    }
  }
  return cudaGetLastError();
}

}  // namespace k
}  // namespace bb
