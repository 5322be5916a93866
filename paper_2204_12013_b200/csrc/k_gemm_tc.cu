// k_gemm_tc.cu — bf16 GEMM on the 5th-generation tensor cores (sm_100a).
//
// D[m][n] = sum_k A(m,k) B(n,k), fp32 accumulation in TMEM, with the fused
// epilogues of kernels.h. One 128 x BN output tile per CTA:
//   warp 0      TMA producer: 64-wide K slabs of A and B, 128B-swizzled, into a
//               `STAGES`-deep shared-memory ring (mbarrier full/empty pairs);
//               K-major operands are one box per slab, MN-major operands are
//               loaded as 64-element MN boxes (UMMA MN-major canonical layout);
//   warp 1      allocates TMEM, one elected lane issues tcgen05.mma
//               (kind::f16, M=128, N=BN, K=16) and tcgen05.commit's the slot
//               back to the producer, then the accumulator to the epilogue;
//   warps 2..5  epilogue: tcgen05.ld 32 columns at a time (warp w reads TMEM
//               lanes 32*(w%4)..+31 = tile rows), apply bias / residual / GELU /
//               GELU' / fp32 accumulate, store.
// Deterministic: every output element is produced by one thread from one
// accumulator whose K order is fixed.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "k_common.cuh"
#include "k_sm100.cuh"

namespace bb {
namespace k {
namespace {
using namespace sm100;

constexpr int BM = 128, BK = 64;
constexpr int kEpiWarps = 8;                 // 2 per TMEM lane quarter
constexpr int kThreads = 64 + 32 * kEpiWarps;

// Instruction descriptor: bf16 x bf16 -> f32, M = 128, N = BN.
__host__ __device__ constexpr uint32_t instr_desc(int n, bool a_mn, bool b_mn, int m) {
  return (1u << 4)                    // D format f32
         | (1u << 7)                  // A bf16
         | (1u << 10)                 // B bf16
         | ((a_mn ? 1u : 0u) << 15)   // A major
         | ((b_mn ? 1u : 0u) << 16)   // B major
         | ((uint32_t)(n >> 3) << 17) // N / 8
         | ((uint32_t)(m >> 4) << 24);
}

// Epilogue over one staged 32-row x 32-column chunk: lane l owns the column
// pair n = n0 + 2(l % 16), n+1 of rows m0 + 2i + l/16 (i < 16), so each warp
// store covers two 64-byte row segments. All row operands are loaded before
// any store so the 16 row loads are in flight together. N, ldc are even
// (gemm_tc_supported), so every pair is fully in or out.
template <int EPI>
__device__ __forceinline__ void epi_chunk(const Gemm &g, const float *stage, int ld_stage, int m0,
                                          int n0, int lane) {
  const int n = n0 + 2 * (lane & 15);
  if (n >= g.N) return;
  const int rsub = lane >> 4;
  float2 b = make_float2(0.f, 0.f);
  if (EPI == EPI_BIAS || EPI == EPI_BIAS_RES || EPI == EPI_BIAS_GELU)
    b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(
        reinterpret_cast<const __nv_bfloat16 *>(g.bias) + n));
  uint32_t pre[16];
  float2 pref[16];
  if (EPI == EPI_BIAS_RES || EPI == EPI_GELU_BWD) {
    const __nv_bfloat16 *src = reinterpret_cast<const __nv_bfloat16 *>(
        EPI == EPI_BIAS_RES ? g.res : g.aux);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int row = m0 + 2 * i + rsub;
      pre[i] = row < g.M ? *reinterpret_cast<const uint32_t *>(src + (size_t)row * g.ldc + n) : 0u;
    }
  }
  if (EPI == EPI_ACC_F32) {
    const float *src = reinterpret_cast<const float *>(g.C);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int row = m0 + 2 * i + rsub;
      pref[i] = row < g.M ? __ldcg(reinterpret_cast<const float2 *>(src + (size_t)row * g.ldc + n))
                          : make_float2(0.f, 0.f);
    }
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int r = 2 * i + rsub, row = m0 + r;
    if (row >= g.M) break;
    const size_t idx = (size_t)row * g.ldc + n;
    const float a0 = stage[r * ld_stage + 2 * (lane & 15)];
    const float a1 = stage[r * ld_stage + 2 * (lane & 15) + 1];
    __nv_bfloat162 *C = reinterpret_cast<__nv_bfloat162 *>(
        reinterpret_cast<__nv_bfloat16 *>(g.C) + idx);
    if (EPI == EPI_STORE) {
      *C = __floats2bfloat162_rn(a0, a1);
    } else if (EPI == EPI_BIAS) {
      *C = __floats2bfloat162_rn(a0 + b.x, a1 + b.y);
    } else if (EPI == EPI_BIAS_RES) {
      const float2 rr = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&pre[i]));
      *C = __floats2bfloat162_rn(a0 + b.x + rr.x, a1 + b.y + rr.y);
    } else if (EPI == EPI_BIAS_GELU) {
      const float p0 = a0 + b.x, p1 = a1 + b.y;
      *reinterpret_cast<__nv_bfloat162 *>(reinterpret_cast<__nv_bfloat16 *>(g.aux) + idx) =
          __floats2bfloat162_rn(p0, p1);
      *C = __floats2bfloat162_rn(gelu_fast(p0), gelu_fast(p1));
    } else if (EPI == EPI_GELU_BWD) {
      const float2 pp = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&pre[i]));
      *C = __floats2bfloat162_rn(a0 * gelu_grad_fast(pp.x), a1 * gelu_grad_fast(pp.y));
    } else if (EPI == EPI_ACC_F32) {
      *reinterpret_cast<float2 *>(reinterpret_cast<float *>(g.C) + idx) =
          make_float2(pref[i].x + a0, pref[i].y + a1);
    } else {   // EPI_STORE_F32
      *reinterpret_cast<float2 *>(reinterpret_cast<float *>(g.C) + idx) = make_float2(a0, a1);
    }
  }
}

// Per-CTA shared memory: a ring of (A, B) K-slabs as deep as fits, the
// epilogue staging and the barriers. With CG = 2 a CTA holds its 128 rows of
// A and half (BN / 2 rows) of B.
template <int BN, int CG, bool TE>
struct Smem {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = (BN / CG) * BK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int EPI_LD = 33;                       // floats per staged row (padded)
  // TE: two 32-row x 128-byte (SW128) boxes per epilogue warp; else the
  // padded fp32 staging of one 32 x 32 chunk per warp.
  static constexpr int EPI_BYTES = TE ? kEpiWarps * 2 * 4096 : kEpiWarps * 32 * EPI_LD * 4;
  static constexpr int BAR_BYTES = 512;
  static constexpr int kMaxSmem = 232448;                 // 227 KB opt-in per CTA
  static constexpr int FIT = (kMaxSmem - EPI_BYTES - 1024 - BAR_BYTES) / STAGE;
  static constexpr int STAGES = FIT > 8 ? 8 : FIT;
  static constexpr int BYTES = STAGES * STAGE + EPI_BYTES + 1024 /*align*/ + BAR_BYTES;
};

// Persistent: CTA b (CTA pair b with CG = 2) processes output tiles b,
// b + grid, ... (N-fastest raster so consecutive CTAs share the A slab in
// L2). Two TMEM accumulators (2 x BN columns) let the epilogue of tile j
// overlap the MMAs of tile j+1.
//
// CG = 2 (cluster of two CTAs on one TPC, tcgen05 cta_group::2): the pair
// computes a 256 x BN tile with M = 256 MMAs issued by CTA 0. CTA r loads
// rows m0 + 128 r of A and rows n0 + r BN/2 of B into its own smem; both
// CTAs' TMA complete on CTA 0's `full` barrier (one arrive + expect_tx for
// both, armed by CTA 0); the MMA commit multicasts `empty` / `tfull` to both
// CTAs; CTA r's epilogue reads its TMEM (= tile rows 128 r ..) and arrives
// on CTA 0's `tempty` (count 2 x kEpiWarps). Each SM fetches 32 KB per
// K slab instead of 48 KB for the same 128 x 256 x 64 MMA work: the mainloop
// is bound by L2 -> SM bandwidth, not by the tensor pipe.
constexpr int tmem_cols(int n) { return n <= 32 ? 32 : n <= 64 ? 64 : n <= 128 ? 128 : n <= 256 ? 256 : 512; }

// BB_GEMM_TRACE: progress words per CTA in mapped host memory (readable by
// the host while a kernel hangs). Word 0 stage (1 running, 2 past the tile
// loops, 3 done), 1/2 producer iteration before / after its empty wait,
// 3/4 MMA iteration waiting for full / tile waiting for tempty, 5/6 epilogue
// tile waiting for tfull / released.
__device__ __forceinline__ void trw(unsigned *t, int i, unsigned v) {
  if (t) *(volatile unsigned *)(t + i) = v;
}

template <int BN, int EPI, int CG, bool TE>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap map_a,
                   const __grid_constant__ CUtensorMap map_b,
                   const __grid_constant__ CUtensorMap map_c,
                   const __grid_constant__ CUtensorMap map_x, Gemm g, int ksplit,
                   int *__restrict__ flags, int epoch) {
  using L = Smem<BN, CG, TE>;
  constexpr int BNH = BN / CG;                     // B rows held by this CTA
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t *gbase = smem_raw + (base - raw);
  float *epi_smem = reinterpret_cast<float *>(gbase + L::STAGES * L::STAGE);
  const uint32_t bars = base + L::STAGES * L::STAGE + L::EPI_BYTES;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (L::STAGES + s); };
  auto tfull_bar = [&](int a) { return bars + 8u * (2 * L::STAGES + a); };
  auto tempty_bar = [&](int a) { return bars + 8u * (2 * L::STAGES + 2 + a); };
  auto in_bar = [&](int w, int b) { return bars + 8u * (2 * L::STAGES + 4 + 2 * w + b); };
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(gbase + L::STAGES * L::STAGE + L::EPI_BYTES +
                                                     8 * (2 * L::STAGES + 4 + 2 * kEpiWarps));

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int rank = CG == 2 ? (int)cluster_ctarank() : 0;
  const int pid = CG == 2 ? (int)cluster_id_x() : blockIdx.x;
  const int npid = CG == 2 ? (int)nclusters_x() : gridDim.x;
  const int nk = (g.K + BK - 1) / BK;
  const int tiles_n = (g.N + BN - 1) / BN, tiles_m = (g.M + BM * CG - 1) / (BM * CG);
  const int tiles = tiles_n * tiles_m;
  // tile -> (row block, column block): N fastest (a wave shares its A rows),
  // or M fastest for wide-N GEMMs whose B is far larger than A (the LM head:
  // a wave then shares B tiles, so the weight is read once, not once per row
  // block). Each tile is still one accumulator over the full K: same bits.
  auto tile_mb = [&](int t) { return g.m_fast ? t % tiles_m : t / tiles_n; };
  auto tile_nb = [&](int t) { return g.m_fast ? t / tiles_m : t % tiles_n; };
  // Work unit = (tile, K split). With ksplit > 1 (fp32-accumulating dW only)
  // the splits of a tile add into C in ascending split order, serialised by a
  // per-(tile, CTA) flag (epoch * 16 + split): deterministic; a split waits
  // only on a lower-numbered CTA of the same round (grid % ksplit == 0).
  const int units = tiles * ksplit;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < L::STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull_bar(a), 1);
      mbar_init(tempty_bar(a), CG * kEpiWarps);   // one arrive per epilogue warp
    }
    if (TE)
      for (int w = 0; w < 2 * kEpiWarps; ++w) mbar_init(in_bar(w / 2, w % 2), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
  }
  if (CG == 2) cluster_sync();          // peer barriers initialised before any remote arrive
  if (warp == 1) {
    if (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "n"(tmem_cols(2 * BN)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "n"(tmem_cols(2 * BN)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  unsigned *tr = g.trace ? g.trace + 8 * blockIdx.x : nullptr;
  if (threadIdx.x == 0) trw(tr, 0, 1);

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs of a pair)
      int it = 0;
      for (int unit = pid; unit < units; unit += npid) {
        const int tile = unit / ksplit, split = unit % ksplit;
        const int kb0 = split * nk / ksplit, kb1 = (split + 1) * nk / ksplit;
        const int m0 = tile_mb(tile) * BM * CG + rank * BM;
        const int nb0 = tile_nb(tile) * BN + rank * BNH;
        // MN-major boxes lying entirely past M (N) are skipped: they only feed
        // output rows (columns) the epilogue masks. Partial boxes are zero-filled.
        // Except: CTA 1 of a pair must load at least one box per K slab. Its
        // bytes are what makes CTA 0's full barrier wait for it; with none
        // (the corner tile of C3's 1600 x 1600 dW: rank 1 past both M and N)
        // the MMA can run STAGES slabs ahead, CTA 1's empty barriers flip
        // twice while its producer lags, its parity wait aliases and the
        // kernel hangs (seen intermittently under concurrent kernels; the
        // round-1 C4 stall). One fully out-of-bounds box (zeros) restores
        // the lockstep.
        auto n_boxes_a_raw = [&](int r) { return max(0, min(BM / 64, (g.M - (m0 + (r - rank) * BM) + 63) / 64)); };
        auto n_boxes_b_raw = [&](int r) { return max(0, min(BNH / 64, (g.N - (nb0 + (r - rank) * BNH) + 63) / 64)); };
        auto dummy = [&](int r) {
          return CG == 2 && r == 1 && g.a_mn && g.b_mn && n_boxes_a_raw(r) == 0 &&
                 n_boxes_b_raw(r) == 0;
        };
        auto n_boxes_a = [&](int r) { return n_boxes_a_raw(r) + (dummy(r) ? 1 : 0); };
        auto n_boxes_b = [&](int r) { return n_boxes_b_raw(r); };
        auto bytes_of = [&](int r) {
          return (uint32_t)((g.a_mn ? n_boxes_a(r) * 64 * BK * 2 : L::A_BYTES) +
                            (g.b_mn ? n_boxes_b(r) * 64 * BK * 2 : L::B_BYTES));
        };
        const int na = g.a_mn ? n_boxes_a(rank) : 1;
        const int nb = g.b_mn ? n_boxes_b(rank) : 1;
        // CTA 0 arms its full barrier for both CTAs' bytes (one arrive); the
        // peer's loads only complete_tx on it (a remote arrive per slab would
        // serialise the peer's producer behind a cluster-scope release).
        const uint32_t bytes = CG == 1 ? bytes_of(0) : bytes_of(0) + bytes_of(1);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % L::STAGES;
          const uint32_t ph = (it / L::STAGES) & 1;
          trw(tr, 1, it + 1);
          mbar_wait(empty_bar(s), ph ^ 1);
          trw(tr, 2, it + 1);
          const uint32_t sa = base + s * L::STAGE, sb = sa + L::A_BYTES;
          const int k0 = kb * BK;
          if (CG == 1) {
            mbar_expect_tx(full_bar(s), bytes);
            if (!g.a_mn) {
              tma_load_2d(sa, &map_a, full_bar(s), k0, m0);
            } else {
              for (int j = 0; j < na; ++j)
                tma_load_2d(sa + j * 64 * BK * 2, &map_a, full_bar(s), m0 + 64 * j, k0);
            }
            if (!g.b_mn) {
              tma_load_2d(sb, &map_b, full_bar(s), k0, nb0);
            } else {
              for (int j = 0; j < nb; ++j)
                tma_load_2d(sb + j * 64 * BK * 2, &map_b, full_bar(s), nb0 + 64 * j, k0);
            }
          } else {
            const uint32_t fb = mapa(full_bar(s), 0);
            if (rank == 0) mbar_expect_tx(full_bar(s), bytes);
            if (!g.a_mn) {
              tma_load_2d_pair(sa, &map_a, fb, k0, m0);
            } else {
              for (int j = 0; j < na; ++j)
                tma_load_2d_pair(sa + j * 64 * BK * 2, &map_a, fb, m0 + 64 * j, k0);
            }
            if (!g.b_mn) {
              tma_load_2d_pair(sb, &map_b, fb, k0, nb0);
            } else {
              for (int j = 0; j < nb; ++j)
                tma_load_2d_pair(sb + j * 64 * BK * 2, &map_b, fb, nb0 + 64 * j, k0);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ---------------- MMA issuer (CTA 0 of a pair)
      const uint32_t idesc = instr_desc(BN, g.a_mn, g.b_mn, BM * CG);
      int it = 0, j = 0;
      for (int unit = pid; unit < units; unit += npid, ++j) {
        const int split = unit % ksplit;
        const int kb0 = split * nk / ksplit, kb1 = (split + 1) * nk / ksplit;
        const int acc = j & 1;
        trw(tr, 4, 0x80000000u | (unsigned)j);
        if (CG == 2) mbar_wait_cluster(tempty_bar(acc), ((j >> 1) & 1) ^ 1);
        else mbar_wait(tempty_bar(acc), ((j >> 1) & 1) ^ 1);
        trw(tr, 4, (unsigned)j);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % L::STAGES;
          const uint32_t ph = (it / L::STAGES) & 1;
          trw(tr, 3, 0x80000000u | (unsigned)it);
          mbar_wait(full_bar(s), ph);
          trw(tr, 3, (unsigned)it);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sa = base + s * L::STAGE, sb = sa + L::A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            // K-major: +32 B per 16-element K step inside the 128B swizzle row;
            // MN-major: +16 rows (2 KB) per K step, 64-element MN chunks 8 KB apart.
            const uint64_t da = g.a_mn ? smem_desc(sa + kk * 2048, 64 * BK * 2, 1024)
                                       : smem_desc(sa + kk * 32, 16, 1024);
            const uint64_t db = g.b_mn ? smem_desc(sb + kk * 2048, 64 * BK * 2, 1024)
                                       : smem_desc(sb + kk * 32, 16, 1024);
            if (CG == 2) mma_bf16_pair(d, da, db, idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
            else mma_bf16(d, da, db, idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
          }
          if (CG == 2) mma_commit_pair(empty_bar(s), 3);
          else mma_commit(empty_bar(s));
        }
        if (CG == 2) mma_commit_pair(tfull_bar(acc), 3);
        else mma_commit(tfull_bar(acc));
      }
    }
  } else if (TE) {
    // ---------------- epilogue, TMA flavour (warps 2..9). Warp w owns tile rows
    // 32 (w % 4).. (its TMEM lane quarter) and one half of the columns, in
    // chunks of 128 bytes per row (64 bf16 / 32 fp32 columns): tcgen05.ld ->
    // fused math -> 128B-swizzled smem box -> one TMA store (or TMA fp32
    // add-reduction for EPI_ACC_F32). Row operands (residual / GELU input) are
    // TMA-loaded into the same box ahead of use, the first chunk's while the
    // tile's MMAs still run. Two boxes per warp alternate so the store of one
    // chunk overlaps the math of the next. TMA clips rows / columns past M / N.
    constexpr bool F32OUT = EPI == EPI_ACC_F32 || EPI == EPI_STORE_F32;
    constexpr int CW = F32OUT ? 32 : 64;
    constexpr bool HAS_IN = EPI == EPI_BIAS_RES || EPI == EPI_GELU_BWD;
    constexpr bool HAS_BIAS = EPI == EPI_BIAS || EPI == EPI_BIAS_RES || EPI == EPI_BIAS_GELU;
    // the tile's BN / CW column chunks alternate between the two warps of a
    // lane quarter (chunk c goes to warp half c % 2)
    constexpr int NCT = BN / CW;
    const int q = warp % 4, half = (warp - 2) / 4, ew = warp - 2;
    const int nch = (NCT - half + 1) / 2;
    const uint32_t box0 = base + L::STAGES * L::STAGE + ew * 8192;
    const uint32_t rowoff = lane * 128;
    const uint32_t my_tempty0 = CG == 2 ? mapa(tempty_bar(0), 0) : tempty_bar(0);
    uint32_t inph = 0;                    // parity bit per box of in_bar
    int bsel = 0;
    int j = 0;
    for (int unit = pid; unit < units; unit += npid, ++j) {
      const int tile = unit / ksplit, split = unit % ksplit;
      const int m0 = tile_mb(tile) * BM * CG + rank * BM, n0 = tile_nb(tile) * BN;
      const int fl = tile * CG + rank;
      const int acc = j & 1;
      const int mr = m0 + q * 32;                         // this warp's first row
      const int nw = n0 + half * CW;                      // this warp's first column
      const bool live = mr < g.M && nw < g.N;
      if (HAS_IN && live && lane == 0) {                  // prefetch chunk 0's row operand
        bulk_wait_read<0>();
        mbar_expect_tx(in_bar(ew, bsel), 4096);
        tma_load_2d(box0 + bsel * 4096, &map_x, in_bar(ew, bsel), nw, mr);
      }
      if (threadIdx.x == 64) trw(tr, 5, 0x80000000u | (unsigned)j);
      mbar_wait(tfull_bar(acc), (j >> 1) & 1);
      if (threadIdx.x == 64) trw(tr, 5, (unsigned)j);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (ksplit > 1 && split > 0) {
        if (threadIdx.x == 64) {
          const volatile int *f = flags + fl;
          while (*f != epoch * 16 + split) __nanosleep(64);
          __threadfence();
          asm volatile("fence.proxy.async;" ::: "memory");
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
      }
#pragma unroll 1
      for (int ch = 0; ch < nch; ++ch) {
        const int n = nw + ch * 2 * CW;
        const bool go = live && n < g.N;
        const int b = bsel;
        if (go) {
          if (lane == 0) {
            if (HAS_IN) {
              if (ch + 1 < nch && n + 2 * CW < g.N) {     // prefetch the next chunk's operand
                bulk_wait_read<0>();
                mbar_expect_tx(in_bar(ew, b ^ 1), 4096);
                tma_load_2d(box0 + (b ^ 1) * 4096, &map_x, in_bar(ew, b ^ 1), n + 2 * CW, mr);
              }
            } else if (EPI == EPI_BIAS_GELU) {
              bulk_wait_read<0>();                        // both boxes are written below
            } else {
              bulk_wait_read<1>();                        // box b's previous store has read it
            }
          }
          __syncwarp();
        }
        uint32_t r0[32], r1[32];
        if (go) {
          const uint32_t t = tmem + acc * BN + ((uint32_t)(q * 32) << 16) + (half + 2 * ch) * CW;
          tmem_ld32_nowait(t, r0);
          if (!F32OUT) tmem_ld32_nowait(t + 32, r1);
          tmem_wait_ld();
          tmem_pin(r0);
          if (!F32OUT) tmem_pin(r1);
        }
        if (ch == nch - 1 || !go) {
          // all TMEM reads of this accumulator done: release it to the MMA warp
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        }
        if (!go) break;
        if (HAS_IN) {
          mbar_wait(in_bar(ew, b), (inph >> b) & 1);
          inph ^= 1u << b;
        }
        const uint32_t box = box0 + b * 4096;
#pragma unroll
        for (int c16 = 0; c16 < 8; ++c16) {               // 16-byte chunk of this lane's row
          const uint32_t addr = box + rowoff + ((c16 ^ (lane & 7)) << 4);
          if (F32OUT) {
            st_shared_v4(addr, r0[4 * c16], r0[4 * c16 + 1], r0[4 * c16 + 2], r0[4 * c16 + 3]);
          } else {
            float x[8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
              x[i] = __uint_as_float(c16 < 4 ? r0[8 * c16 + i] : r1[8 * (c16 - 4) + i]);
            if (HAS_BIAS) {
              const int nb = n + 8 * c16;
#pragma unroll
              for (int i = 0; i < 8; i += 2) {
                float2 bv = make_float2(0.f, 0.f);
                if (nb + i < g.N)
                  bv = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(
                      reinterpret_cast<const __nv_bfloat16 *>(g.bias) + nb + i));
                x[i] += bv.x;
                x[i + 1] += bv.y;
              }
            }
            uint32_t o[4];
            if (HAS_IN) {
              const uint4 in = ld_shared_v4(addr);
              const uint32_t iw[4] = {in.x, in.y, in.z, in.w};
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float2 p = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&iw[i]));
                float y0, y1;
                if (EPI == EPI_BIAS_RES) {
                  y0 = x[2 * i] + p.x;
                  y1 = x[2 * i + 1] + p.y;
                } else {
                  y0 = x[2 * i] * gelu_grad_fast(p.x);
                  y1 = x[2 * i + 1] * gelu_grad_fast(p.y);
                }
                __nv_bfloat162 h = __floats2bfloat162_rn(y0, y1);
                o[i] = *reinterpret_cast<uint32_t *>(&h);
              }
            } else if (EPI == EPI_BIAS_GELU) {
              uint32_t pa[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                __nv_bfloat162 hp = __floats2bfloat162_rn(x[2 * i], x[2 * i + 1]);
                pa[i] = *reinterpret_cast<uint32_t *>(&hp);
                __nv_bfloat162 h = __floats2bfloat162_rn(gelu_fast(x[2 * i]), gelu_fast(x[2 * i + 1]));
                o[i] = *reinterpret_cast<uint32_t *>(&h);
              }
              st_shared_v4(box0 + (b ^ 1) * 4096 + rowoff + ((c16 ^ (lane & 7)) << 4), pa[0], pa[1],
                           pa[2], pa[3]);
            } else {
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                __nv_bfloat162 h = __floats2bfloat162_rn(x[2 * i], x[2 * i + 1]);
                o[i] = *reinterpret_cast<uint32_t *>(&h);
              }
            }
            st_shared_v4(addr, o[0], o[1], o[2], o[3]);
          }
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          if (EPI == EPI_ACC_F32) tma_reduce_add_2d(&map_c, box, n, mr);
          else tma_store_2d(&map_c, box, n, mr);
          if (EPI == EPI_BIAS_GELU) tma_store_2d(&map_x, box0 + (b ^ 1) * 4096, n, mr);
          bulk_commit();
        }
        bsel ^= 1;
      }
      if (lane == 0) {
        if (CG == 2) mbar_arrive_cluster(my_tempty0 + 8u * acc);
        else mbar_arrive(tempty_bar(acc));
      }
      if (threadIdx.x == 64) trw(tr, 6, (unsigned)j + 1);
      if (ksplit > 1) {
        if (lane == 0) {
          bulk_wait<0>();                                 // this warp's adds are performed
          asm volatile("fence.proxy.async;" ::: "memory");
          __threadfence();
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
        if (threadIdx.x == 64) *(volatile int *)(flags + fl) = epoch * 16 + split + 1;
      }
    }
    if (lane == 0) bulk_wait<0>();                        // smem boxes read before exit
  } else {
    // ---------------- epilogue, LSU flavour (warps 2..9): TMEM -> regs -> smem -> coalesced rows
    const int q = warp % 4;               // TMEM lane quarter this warp may read
    const int half = (warp - 2) / 4;      // which half of the tile's columns
    float *stage = epi_smem + (warp - 2) * 32 * L::EPI_LD;
    const uint32_t my_tempty0 = CG == 2 ? mapa(tempty_bar(0), 0) : tempty_bar(0);
    int j = 0;
    for (int unit = pid; unit < units; unit += npid, ++j) {
      const int tile = unit / ksplit, split = unit % ksplit;
      const int m0 = tile_mb(tile) * BM * CG + rank * BM, n0 = tile_nb(tile) * BN;
      const int fl = tile * CG + rank;
      const int acc = j & 1;
      mbar_wait(tfull_bar(acc), (j >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (ksplit > 1 && split > 0) {
        if (threadIdx.x == 64) {
          const volatile int *f = flags + fl;
          while (*f != epoch * 16 + split) __nanosleep(64);
          __threadfence();
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
      }
      const int ncols = m0 < g.M ? min(BN, g.N - n0) : 0;
#pragma unroll 1
      for (int c = half * (BN / 2); c < min(ncols, (half + 1) * (BN / 2)); c += 32) {
        float v[32];
        tmem_ld32(tmem + acc * BN + ((uint32_t)(q * 32) << 16) + c, v);
#pragma unroll
        for (int i = 0; i < 32; ++i) stage[lane * L::EPI_LD + i] = v[i];
        __syncwarp();
        epi_chunk<EPI>(g, stage, L::EPI_LD, m0 + q * 32, n0 + c, lane);
        __syncwarp();
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      if (lane == 0) {
        if (CG == 2) mbar_arrive_cluster(my_tempty0 + 8u * acc);
        else mbar_arrive(tempty_bar(acc));
      }
      if (ksplit > 1) {
        __threadfence();
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
        if (threadIdx.x == 64) *(volatile int *)(flags + fl) = epoch * 16 + split + 1;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) trw(tr, 0, 2);
  if (CG == 2) cluster_sync();          // peer MMAs / remote arrives done before dealloc / exit
  if (threadIdx.x == 0) trw(tr, 0, 3);
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (CG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(tmem_cols(2 * BN)));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(tmem_cols(2 * BN)));
  }
}

// ------------------------------------------------------------------ host
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2D bf16 tensor map: inner dimension `inner` (contiguous), `outer` rows of
// `ld` elements, box {64, box_outer}, 128B swizzle, zero OOB fill.
bool make_map(CUtensorMap *m, const void *ptr, uint64_t inner, uint64_t outer, uint64_t ld,
              uint32_t box_outer) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {64, box_outer};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Epilogue box map: {inner, outer} elements of `es` bytes, row pitch ld
// elements, box {128 / es, 32}, 128B swizzle (the epilogue's smem box layout).
bool make_epi_map(CUtensorMap *m, const void *ptr, bool f32, uint64_t inner, uint64_t outer,
                  uint64_t ld) {
  auto fn = encode_fn();
  if (!fn) return false;
  const uint64_t es = f32 ? 4 : 2;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * es};
  cuuint32_t box[2] = {(cuuint32_t)(128 / es), 32};
  cuuint32_t el[2] = {1, 1};
  return fn(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
            const_cast<void *>(ptr), dims, strides, box, el, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Per-launch slice of a device flag ring for serialised split-K; every launch
// gets a fresh epoch, so flags never need resetting.
int *split_flags(int n, int *epoch) {
  static std::mutex mu;
  static int *ring = nullptr;
  static int cursor = 0, ep = 0;
  constexpr int kRing = 1 << 20;
  std::lock_guard<std::mutex> lk(mu);
  if (!ring) {
    if (cudaMalloc(&ring, kRing * sizeof(int)) != cudaSuccess) return nullptr;
    // legacy-stream memset, then a device sync: the flags are read by
    // kernels on non-blocking streams
    if (cudaMemset(ring, 0, kRing * sizeof(int)) != cudaSuccess) return nullptr;
    if (cudaDeviceSynchronize() != cudaSuccess) return nullptr;
  }
  if (cursor + n > kRing) cursor = 0;
  int *p = ring + cursor;
  cursor += n;
  ep = (ep + 1) & ((1 << 26) - 1);
  if (ep == 0) ep = 1;
  *epoch = ep;
  return p;
}

int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return sms;
}

// ---- BB_GEMM_TRACE ring: one region of per-CTA words per launch
constexpr int kTrLaunches = 2048, kTrCtas = 296;
struct TraceRec { int M, N, K, epi, bn, cg, grid, ksplit; };
unsigned *g_tr_host = nullptr, *g_tr_dev = nullptr;
TraceRec g_tr_rec[kTrLaunches];
long long g_tr_n = 0;
std::mutex g_tr_mu;
unsigned *trace_slot(const Gemm &g, int bn, int cg, int grid, int ksplit) {
  static const bool on = std::getenv("BB_GEMM_TRACE") != nullptr;
  if (!on || grid > kTrCtas) return nullptr;
  std::lock_guard<std::mutex> lk(g_tr_mu);
  if (!g_tr_host) {
    const size_t bytes = (size_t)kTrLaunches * kTrCtas * 8 * 4;
    if (cudaHostAlloc(&g_tr_host, bytes, cudaHostAllocMapped) != cudaSuccess) return nullptr;
    std::memset(g_tr_host, 0, bytes);
    if (cudaHostGetDevicePointer(&g_tr_dev, g_tr_host, 0) != cudaSuccess) return nullptr;
  }
  const int i = (int)(g_tr_n++ % kTrLaunches);
  std::memset(g_tr_host + (size_t)i * kTrCtas * 8, 0, kTrCtas * 8 * 4);
  g_tr_rec[i] = {g.M, g.N, g.K, g.epi, bn, cg, grid, ksplit};
  return g_tr_dev + (size_t)i * kTrCtas * 8;
}

template <int BN, int EPI, int CG, bool TE>
cudaError_t launch(const Gemm &g_in, cudaStream_t s) {
  Gemm g = g_in;
  // M-fastest tile order when B (N x K) is several times A and too big to
  // stay in L2 across row blocks (measured: the C3 LM-head forward read its
  // 161 MB weight 16 times, 2.9 GB per launch, profiles/r02_gemm_shapes_c3.json)
  g.m_fast = (long long)g.N >= 4LL * g.M && (long long)g.N * g.K * 2 > (64LL << 20);
  constexpr int BNH = BN / CG;
  using L = Smem<BN, CG, TE>;
  auto kern = gemm_tc_kernel<BN, EPI, CG, TE>;
  CUtensorMap ma, mb, mc, mx;
  // K-major operand: tensor {K, rows}, box {64, tile rows}; MN-major: tensor {rows, K}, box {64, 64}
  const bool ok_a = g.a_mn ? make_map(&ma, g.A, g.M, g.K, g.lda, BK)
                           : make_map(&ma, g.A, g.K, g.M, g.lda, BM);
  const bool ok_b = g.b_mn ? make_map(&mb, g.B, g.N, g.K, g.ldb, BK)
                           : make_map(&mb, g.B, g.K, g.N, g.ldb, BNH);
  if (!ok_a || !ok_b) return cudaErrorInvalidValue;
  constexpr bool F32OUT = EPI == EPI_ACC_F32 || EPI == EPI_STORE_F32;
  if (TE) {
    if (!make_epi_map(&mc, g.C, F32OUT, g.N, g.M, g.ldc)) return cudaErrorInvalidValue;
    const void *x = EPI == EPI_BIAS_RES ? g.res : g.aux;
    if (EPI == EPI_BIAS_RES || EPI == EPI_GELU_BWD || EPI == EPI_BIAS_GELU) {
      if (!make_epi_map(&mx, x, false, g.N, g.M, g.ldc)) return cudaErrorInvalidValue;
    } else {
      mx = mc;
    }
  } else {
    mc = ma;
    mx = ma;
  }
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         L::BYTES);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int tiles = ((g.N + BN - 1) / BN) * ((g.M + BM * CG - 1) / (BM * CG));
  // Resident CTAs (pairs): a pair needs both SMs of one TPC free, and not
  // every TPC has two usable SMs, so ask the occupancy calculator.
  static int slots = 0;
  if (!slots) {
    slots = num_sms() / CG;
    if (CG > 1) {
      cudaLaunchConfig_t oc = {};
      oc.gridDim = dim3(CG * slots);
      oc.blockDim = dim3(kThreads);
      oc.dynamicSmemBytes = L::BYTES;
      cudaLaunchAttribute at;
      at.id = cudaLaunchAttributeClusterDimension;
      at.val.clusterDim.x = CG;
      at.val.clusterDim.y = 1;
      at.val.clusterDim.z = 1;
      oc.attrs = &at;
      oc.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, kern, &oc) == cudaSuccess &&
          n > 0)
        slots = std::min(slots, n);
      if (std::getenv("BB_DEBUG")) fprintf(stderr, "[bb] gemm pair slots %d\n", slots);
    }
  }
  // Split K for fp32-accumulating GEMMs (dW) whose tiles cannot fill the GPU
  // twice over. (A general rounds-minimising split count was measured slower
  // at C3: the serialised split adds cost more than the quantisation they
  // remove, gemm_dw 476 -> 642 ms per serialised step.)
  const int nk = (g.K + BK - 1) / BK;
  int ksplit = 1;
  if (EPI == EPI_ACC_F32 && tiles * 2 <= slots && !g.tile_grid)
    ksplit = std::max(1, std::min({slots / tiles, nk / 8, 8}));
  int *flags = nullptr;
  int epoch = 0;
  if (ksplit > 1) {
    flags = split_flags(tiles * CG, &epoch);
    if (!flags) ksplit = 1;
  }
  const int units = tiles * ksplit;
  // Split-K waits only on the previous split of the same tile. With the number
  // of persistent CTAs (pairs) a multiple of ksplit, every round covers whole
  // tiles, so that split always runs on a lower-numbered CTA in the same
  // round: dispatched earlier, hence resident, even when other kernels share
  // the GPU and this grid is only partly resident (no co-residency assumed).
  int pids = units < slots || g.tile_grid ? units : slots;
  if (ksplit > 1) pids = std::max(ksplit, pids / ksplit * ksplit);
  const int grid = pids * CG;
  g.trace = trace_slot(g, BN, CG, grid, ksplit);
  if (CG == 1) {
    kern<<<grid, kThreads, L::BYTES, s>>>(ma, mb, mc, mx, g, ksplit, flags, epoch);
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = L::BYTES;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CG;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ma, mb, mc, mx, g, ksplit, flags, epoch);
    if (e != cudaSuccess) return e;
  }
  ++g_launches;
  return cudaGetLastError();
}
}  // namespace

bool tma_map_bf16_2d(CUtensorMap *m, const void *ptr, uint64_t inner, uint64_t outer, uint64_t ld,
                     uint32_t box_outer) {
  return make_map(m, ptr, inner, outer, ld, box_outer);
}

bool tma_map_3d(CUtensorMap *m, const void *ptr, bool f32, const uint64_t dims[3],
                const uint64_t strides_bytes[2], const uint32_t box[3]) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t d[3] = {dims[0], dims[1], dims[2]};
  cuuint64_t st[2] = {strides_bytes[0], strides_bytes[1]};
  cuuint32_t bx[3] = {box[0], box[1], box[2]};
  cuuint32_t el[3] = {1, 1, 1};
  return fn(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
            const_cast<void *>(ptr), d, st, bx, el, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool gemm_tc_supported(const Gemm &g) {
  if (g.M < 1 || g.N < 1 || g.K < 1) return false;
  if ((reinterpret_cast<uintptr_t>(g.A) | reinterpret_cast<uintptr_t>(g.B)) & 15) return false;
  if (g.lda % 8 || g.ldb % 8 || g.N % 2 || g.ldc % 2) return false;
  if (g.epi < EPI_STORE || g.epi > EPI_STORE_F32) return false;
  // MN-major operands need at least one 64-wide box along M / N
  if ((g.a_mn && g.M < 64) || (g.b_mn && g.N < 64)) return false;
  return encode_fn() != nullptr;
}

template <int BN, int CG, bool TE>
cudaError_t launch_bn(const Gemm &g, cudaStream_t s) {
  switch (g.epi) {
    case EPI_STORE: return launch<BN, EPI_STORE, CG, TE>(g, s);
    case EPI_BIAS: return launch<BN, EPI_BIAS, CG, TE>(g, s);
    case EPI_BIAS_RES: return launch<BN, EPI_BIAS_RES, CG, TE>(g, s);
    case EPI_BIAS_GELU: return launch<BN, EPI_BIAS_GELU, CG, TE>(g, s);
    case EPI_GELU_BWD: return launch<BN, EPI_GELU_BWD, CG, TE>(g, s);
    case EPI_ACC_F32: return launch<BN, EPI_ACC_F32, CG, TE>(g, s);
    default: return launch<BN, EPI_STORE_F32, CG, TE>(g, s);
  }
}

// The TMA epilogue needs 16-byte aligned C / residual / aux bases and row
// pitches (tensor-map rules); anything else takes the LSU epilogue.
bool tma_epilogue_ok(const Gemm &g) {
  const bool f32 = g.epi == EPI_ACC_F32 || g.epi == EPI_STORE_F32;
  const uintptr_t mask = reinterpret_cast<uintptr_t>(g.C) |
                         (g.epi == EPI_BIAS_RES ? reinterpret_cast<uintptr_t>(g.res) : 0) |
                         (g.epi == EPI_BIAS_GELU || g.epi == EPI_GELU_BWD
                              ? reinterpret_cast<uintptr_t>(g.aux) : 0);
  if (mask & 15) return false;
  return ((size_t)g.ldc * (f32 ? 4 : 2)) % 16 == 0;
}

// Tile choice. Default: 256 x 256 tiles on CTA pairs with the TMA epilogue
// whenever N >= 256 and the epilogue operands are 16-byte aligned (the
// mainloop is L2 / smem bandwidth bound, so halving each SM's operand
// traffic is what raises the tensor-pipe duty cycle); otherwise single-CTA
// 128 x 256 / 128 x 128 tiles. BB_GEMM_TILE=pair|256|128 and BB_GEMM_EPI=lsu
// force a kind (experiments / tests).
cudaError_t gemm_tc(const Gemm &g, cudaStream_t s) {
  static const int force = [] {
    const char *e = std::getenv("BB_GEMM_TILE");
    if (!e) return 0;
    if (!std::strcmp(e, "pair")) return 2;
    if (!std::strcmp(e, "pair128")) return 3;
    if (!std::strcmp(e, "pair192")) return 4;
    if (!std::strcmp(e, "256")) return 256;
    if (!std::strcmp(e, "128")) return 128;
    return 0;
  }();
  static const bool lsu = [] {
    const char *e = std::getenv("BB_GEMM_EPI");
    return e && !std::strcmp(e, "lsu");
  }();
  const bool te = !lsu && tma_epilogue_ok(g);
  if (force == 128 || g.N < 256)
    return te ? launch_bn<128, 1, true>(g, s) : launch_bn<128, 1, false>(g, s);
  if (force == 256) return te ? launch_bn<256, 1, true>(g, s) : launch_bn<256, 1, false>(g, s);
  if (force == 3 && te) return launch_bn<128, 2, true>(g, s);
  // 256 x 192 pair tiles (K-major B only: 96 B rows per CTA; ragged N is
  // clipped by TMA): fewer tile rounds at N = 768 / 1600, but per flop they
  // move ~17% more operand bytes, and measured no faster (C1: 18.7 vs 18.9 us;
  // C3 step: gemm_fwd 828 vs 819 ms serialised), so only on request
  // (BB_GEMM_TILE=pair192).
  if (force == 4 && te && !g.b_mn && g.epi != EPI_ACC_F32) return launch_bn<192, 2, true>(g, s);
  if (!te) return launch_bn<256, 1, false>(g, s);
  // fp32-accumulating dW with few output tiles: the serialised split-K chain
  // (up to 8 links of a few us each on pairs) costs more than the smaller
  // tiles' lower rate, so take 128 x 128 tiles (shorter chains) there.
  if (force != 2 && g.epi == EPI_ACC_F32 &&
      (long)((g.M + 255) / 256) * ((g.N + 255) / 256) < 16)
    return launch_bn<128, 1, true>(g, s);
  return launch_bn<256, 2, true>(g, s);
}

void gemm_trace_dump() {
  if (!g_tr_host) return;
  const long long n = g_tr_n;
  for (long long l = std::max(0LL, n - kTrLaunches); l < n; ++l) {
    const int i = (int)(l % kTrLaunches);
    const TraceRec &r = g_tr_rec[i];
    const unsigned *t = g_tr_host + (size_t)i * kTrCtas * 8;
    int unfinished = 0;
    for (int c = 0; c < r.grid; ++c) unfinished += t[8 * c] != 3;
    if (!unfinished) continue;
    std::fprintf(stderr, "[bb] gemm launch %lld: %dx%dx%d epi %d BN %d CG %d grid %d ksplit %d, "
                 "%d CTAs unfinished:\n", l, r.M, r.N, r.K, r.epi, r.bn, r.cg, r.grid, r.ksplit,
                 unfinished);
    for (int c = 0; c < r.grid; ++c)
      if (t[8 * c] != 3)
        std::fprintf(stderr, "  cta %d: st %u prod %u/%u mma full %x tempty %x epi tfull %x rel %u\n", c,
                     t[8 * c], t[8 * c + 1], t[8 * c + 2], t[8 * c + 3], t[8 * c + 4], t[8 * c + 5],
                     t[8 * c + 6]);
  }
}

}  // namespace k
}  // namespace bb
