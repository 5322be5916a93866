// k_attn_umma.cu — flash attention forward on the 5th-generation tensor cores
// (tcgen05 / TMEM / TMA), head dim 64, bf16 in, fp32 accumulation.
//
// One CTA = 128 query rows of one (sequence, head); key blocks of 128.
//   warp 0      TMA: the Q tile once, then K_j and V_j into a 2-stage ring
//               (128B-swizzled, straight out of the packed [B*S, 3H] qkv);
//   warp 1      allocates 512 TMEM columns and issues, in order,
//               S_{j+1} = Q K_{j+1}^T (M=128, N=128, K=64, into S buffer
//               (j+1)%2) and, once the softmax published P_j,
//               O += P_j V_j (M=128, N=64, K=128; V is the MN-major B operand);
//   warps 2..5  softmax: thread r owns query row r (TMEM lane r), reads its S
//               row from TMEM, keeps the running max / sum in registers,
//               rescales its O row in TMEM (after PV_{j-1} completed), writes
//               P_j (bf16) into the 128B-swizzled K-major smem tile the next
//               MMA reads, and at the end normalises O and stores O and LSE.
// Same math and LSE convention as the mma.sync kernel (k_attn_tc.cu), used
// for the backward pass.
#include "k_common.cuh"
#include "k_sm100.cuh"

namespace bb {
namespace k {
namespace {
using namespace sm100;

constexpr int D = 64, BQ = 128, BKV = 128, ST = 2;
constexpr int kThreads = 192;
constexpr float LOG2E = 1.4426950408889634f;

constexpr uint32_t idesc_f16(int m, int n, bool a_mn, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

struct SmemLayout {
  static constexpr int Q = 0;                         // 128 x 64 bf16 = 16 KB
  static constexpr int K = Q + BQ * D * 2;            // ST x 16 KB
  static constexpr int V = K + ST * BKV * D * 2;      // ST x 16 KB
  static constexpr int P = V + ST * BKV * D * 2;      // 128 x 128 bf16 = 32 KB (2 swizzle atoms)
  static constexpr int BAR = P + BQ * BKV * 2;
  static constexpr int BYTES = BAR + 256 + 1024;
};

__global__ void __launch_bounds__(kThreads, 1)
    fa_fwd_umma_kernel(const __grid_constant__ CUtensorMap map_qkv, int S, int H, int nh,
                       int causal, __nv_bfloat16 *__restrict__ o, float *__restrict__ lse) {
  using L = SmemLayout;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t *gbase = smem_raw + (base - raw);
  const uint32_t bars = base + L::BAR;
  const uint32_t q_full = bars;
  auto kv_full = [&](int s) { return bars + 8u * (1 + s); };
  auto kv_empty = [&](int s) { return bars + 8u * (1 + ST + s); };
  auto s_full = [&](int b) { return bars + 8u * (1 + 2 * ST + b); };
  const uint32_t p_full = bars + 8u * (3 + 2 * ST);
  const uint32_t o_done = bars + 8u * (4 + 2 * ST);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(gbase + L::BAR + 8 * (5 + 2 * ST));

  const int qb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int q0 = qb * BQ;
  const int row_base = b * S;            // first qkv row of this sequence
  const int nkb_all = (S + BKV - 1) / BKV;
  const int nkb = causal ? min(nkb_all, (q0 + BQ - 1) / BKV + 1) : nkb_all;

  if (warp == 0 && lane == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < ST; ++s) {
      mbar_init(kv_full(s), 1);
      mbar_init(kv_empty(s), 1);
    }
    mbar_init(s_full(0), 1);
    mbar_init(s_full(1), 1);
    mbar_init(p_full, 4);     // one arrive per softmax warp
    mbar_init(o_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_qkv)) : "memory");
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
  const uint32_t t_s[2] = {tmem, tmem + 128};
  const uint32_t t_o = tmem + 256;

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(q_full, BQ * D * 2);
      tma_load_2d(base + L::Q, &map_qkv, q_full, h * D, row_base + q0);
      for (int j = 0; j < nkb; ++j) {
        const int s = j % ST;
        mbar_wait(kv_empty(s), ((j / ST) & 1) ^ 1);
        mbar_expect_tx(kv_full(s), 2 * BKV * D * 2);
        tma_load_2d(base + L::K + s * BKV * D * 2, &map_qkv, kv_full(s), H + h * D,
                    row_base + j * BKV);
        tma_load_2d(base + L::V + s * BKV * D * 2, &map_qkv, kv_full(s), 2 * H + h * D,
                    row_base + j * BKV);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t id_s = idesc_f16(128, BKV, false, false);
      const uint32_t id_o = idesc_f16(128, D, false, true);
      auto issue_s = [&](int j) {
        const int s = j % ST;
        mbar_wait(kv_full(s), (j / ST) & 1);
        tc_fence_after();
        const uint32_t ka = base + L::K + s * BKV * D * 2;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_bf16(t_s[j & 1], smem_desc(base + L::Q + kk * 32, 16, 1024),
                   smem_desc(ka + kk * 32, 16, 1024), id_s, kk > 0 ? 1u : 0u);
        mma_commit(s_full(j & 1));
      };
      mbar_wait(q_full, 0);
      tc_fence_after();
      issue_s(0);
      for (int j = 0; j < nkb; ++j) {
        if (j + 1 < nkb) issue_s(j + 1);
        mbar_wait(p_full, j & 1);
        tc_fence_after();
        const int s = j % ST;
        const uint32_t va = base + L::V + s * BKV * D * 2;
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk) {
          // P: K-major, two 64-key swizzle atoms (16 KB apart); V: MN-major,
          // 16 keys = 16 rows of 128 B per K step.
          const uint64_t da = smem_desc(base + L::P + (kk / 4) * (BQ * 64 * 2) + (kk % 4) * 32, 16,
                                        1024);
          const uint64_t db = smem_desc(va + kk * 2048, 8192, 1024);
          mma_bf16(t_o, da, db, id_o, (j > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(o_done);
        mma_commit(kv_empty(s));
      }
    }
  } else {
    // ---------------- softmax warps: row r = query q0 + r, TMEM lane r
    const int r = (warp % 4) * 32 + lane;
    const int qrow = q0 + r;
    const uint32_t lane_off = (uint32_t)((warp % 4) * 32) << 16;
    const float sl2 = rsqrtf((float)D) * LOG2E;
    float m = -INFINITY, l = 0.f;
    uint8_t *prow = gbase + L::P + r * 128;   // atom 0 row r; atom 1 at +16 KB
    for (int j = 0; j < nkb; ++j) {
      mbar_wait(s_full(j & 1), (j >> 1) & 1);
      tc_fence_after();
      float sv[BKV];
#pragma unroll
      for (int c = 0; c < BKV / 32; ++c) {
        float t[32];
        tmem_ld32(t_s[j & 1] + lane_off + c * 32, t);
#pragma unroll
        for (int i = 0; i < 32; ++i) sv[c * 32 + i] = t[i] * sl2;
      }
      const bool need_mask = (j * BKV + BKV > S) || (causal && j * BKV + BKV - 1 > q0);
      if (need_mask) {
#pragma unroll
        for (int i = 0; i < BKV; ++i) {
          const int key = j * BKV + i;
          if (key >= S || (causal && key > qrow)) sv[i] = -INFINITY;
        }
      }
      float mb = -INFINITY;
#pragma unroll
      for (int i = 0; i < BKV; ++i) mb = fmaxf(mb, sv[i]);
      const float mn = fmaxf(m, mb);
      const float corr = mn == -INFINITY ? 1.f : exp2f(m - mn);
      m = mn;
      float sum = 0.f;
#pragma unroll
      for (int i = 0; i < BKV; ++i) {
        const float p = mn == -INFINITY ? 0.f : exp2f(sv[i] - mn);
        sv[i] = p;
        sum += p;
      }
      l = l * corr + sum;
      if (j > 0) {
        mbar_wait(o_done, (j - 1) & 1);    // PV_{j-1} done: O stable, P buffer free
        tc_fence_after();
        if (__any_sync(0xffffffffu, corr != 1.f)) {
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            float t[32];
            tmem_ld32(t_o + lane_off + c * 32, t);
#pragma unroll
            for (int i = 0; i < 32; ++i) t[i] *= corr;
            tmem_st32(t_o + lane_off + c * 32, t);
          }
        }
      }
      // P row -> swizzled K-major smem (chunk c of 8 keys at position c ^ (r & 7))
#pragma unroll
      for (int c = 0; c < BKV / 8; ++c) {
        uint4 u;
        u.x = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(sv[8 * c])) |
              ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(sv[8 * c + 1])) << 16);
        u.y = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(sv[8 * c + 2])) |
              ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(sv[8 * c + 3])) << 16);
        u.z = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(sv[8 * c + 4])) |
              ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(sv[8 * c + 5])) << 16);
        u.w = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(sv[8 * c + 6])) |
              ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(sv[8 * c + 7])) << 16);
        const int atom = c / 8, cc = c % 8;
        *reinterpret_cast<uint4 *>(prow + atom * (BQ * 64 * 2) + ((cc ^ (r & 7)) * 16)) = u;
      }
      fence_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
    }
    mbar_wait(o_done, (nkb - 1) & 1);
    tc_fence_after();
    float ov[D];
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      float t[32];
      tmem_ld32(t_o + lane_off + c * 32, t);
#pragma unroll
      for (int i = 0; i < 32; ++i) ov[c * 32 + i] = t[i];
    }
    if (qrow < S) {
      const float inv = 1.f / l;
      __nv_bfloat16 *orow = o + ((size_t)row_base + qrow) * H + h * D;
#pragma unroll
      for (int c = 0; c < D / 8; ++c) {
        uint4 u;
        __nv_bfloat162 *hv = reinterpret_cast<__nv_bfloat162 *>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          hv[i] = __floats2bfloat162_rn(ov[8 * c + 2 * i] * inv, ov[8 * c + 2 * i + 1] * inv);
        *reinterpret_cast<uint4 *>(orow + 8 * c) = u;
      }
      lse[((size_t)b * nh + h) * S + qrow] = (m + log2f(l)) / LOG2E;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
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
  dim3 grid((S + BQ - 1) / BQ, nh, B);
  fa_fwd_umma_kernel<<<grid, kThreads, SmemLayout::BYTES, s>>>(
      map, S, H, nh, causal ? 1 : 0, reinterpret_cast<__nv_bfloat16 *>(o), lse);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace k
}  // namespace bb
