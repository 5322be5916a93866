// k_attn_simt.cu — exact-fp32 (SIMT) scaled-dot-product attention forward and
// deterministic backward, per (sequence, head). Used by the fp32 check mode
// and for head dims the tensor-core kernel does not cover.
//
// Forward: o_i = sum_j softmax_j(q_i.k_j/sqrt(d) + mask) v_j, lse_i saved.
// Backward (no atomics): D_i = do_i.o_i; kernel A per query row computes dq_i;
// kernel B per key row computes dk_j, dv_j by looping over the queries.
#include "k_common.cuh"

namespace bb {
namespace k {
namespace {
constexpr int DMAX = 64;
constexpr int WPB = 4;   // warps (rows) per block

// One warp per query row; lane l handles keys j = l, l+32, ...
template <typename T>
__global__ void attn_fwd_kernel(int S, int H, int nh, int causal, const T *__restrict__ qkv,
                                T *__restrict__ o, float *__restrict__ lse) {
  const int d = H / nh;
  const int lane = threadIdx.x % 32, wid = threadIdx.x / 32;
  const int i = blockIdx.x * WPB + wid;
  const int h = blockIdx.y, b = blockIdx.z;
  __shared__ float qs[WPB][DMAX];
  if (i >= S) return;
  const size_t ld = 3 * (size_t)H;
  const T *Q = qkv + ((size_t)b * S) * ld + h * d;
  const T *K = Q + H;
  const T *Vv = Q + 2 * H;
  const float scale = rsqrtf((float)d);
  for (int c = lane; c < d; c += 32) qs[wid][c] = to_f(Q[(size_t)i * ld + c]) * scale;
  __syncwarp();
  float m = -INFINITY, l = 0.f, acc[DMAX];
#pragma unroll
  for (int c = 0; c < DMAX; ++c) acc[c] = 0.f;
  const int jend = causal ? i + 1 : S;
  for (int j = lane; j < jend; j += 32) {
    const T *kr = K + (size_t)j * ld;
    float sc = 0.f;
    for (int c = 0; c < d; ++c) sc = fmaf(qs[wid][c], to_f(kr[c]), sc);
    const float mn = fmaxf(m, sc);
    const float corr = __expf(m - mn), p = __expf(sc - mn);
    l = l * corr + p;
    const T *vr = Vv + (size_t)j * ld;
#pragma unroll
    for (int c = 0; c < DMAX; ++c)
      if (c < d) acc[c] = acc[c] * corr + p * to_f(vr[c]);
    m = mn;
  }
  const float M = warp_max(m);
  const float f = (m == -INFINITY) ? 0.f : __expf(m - M);
  const float L = warp_sum(l * f);
  T *orow = o + ((size_t)b * S + i) * H + h * d;
#pragma unroll
  for (int c = 0; c < DMAX; ++c) {
    if (c < d) {
      const float v = warp_sum(acc[c] * f);
      if (lane == (c % 32)) orow[c] = from_f<T>(v / L);
    }
  }
  if (lane == 0) lse[((size_t)b * nh + h) * S + i] = M + logf(L);
}

// D_i = do_i . o_i
template <typename T>
__global__ void attn_bwd_d_kernel(int S, int H, int nh, const T *__restrict__ o,
                                  const T *__restrict__ dout, float *__restrict__ Dv) {
  const int d = H / nh;
  const int lane = threadIdx.x % 32, wid = threadIdx.x / 32;
  const int i = blockIdx.x * WPB + wid;
  const int h = blockIdx.y, b = blockIdx.z;
  if (i >= S) return;
  const size_t off = ((size_t)b * S + i) * H + h * d;
  float s = 0.f;
  for (int c = lane; c < d; c += 32) s += to_f(o[off + c]) * to_f(dout[off + c]);
  s = warp_sum(s);
  if (lane == 0) Dv[((size_t)b * nh + h) * S + i] = s;
}

template <typename T>
__global__ void attn_bwd_dq_kernel(int S, int H, int nh, int causal, const T *__restrict__ qkv,
                                   const float *__restrict__ lse, const T *__restrict__ dout,
                                   const float *__restrict__ Dv, T *__restrict__ dqkv) {
  const int d = H / nh;
  const int lane = threadIdx.x % 32, wid = threadIdx.x / 32;
  const int i = blockIdx.x * WPB + wid;
  const int h = blockIdx.y, b = blockIdx.z;
  __shared__ float qs[WPB][DMAX], dos[WPB][DMAX];
  if (i >= S) return;
  const size_t ld = 3 * (size_t)H;
  const T *Q = qkv + ((size_t)b * S) * ld + h * d;
  const T *K = Q + H;
  const T *Vv = Q + 2 * H;
  const float scale = rsqrtf((float)d);
  const size_t orow = ((size_t)b * S + i) * H + h * d;
  for (int c = lane; c < d; c += 32) {
    qs[wid][c] = to_f(Q[(size_t)i * ld + c]) * scale;
    dos[wid][c] = to_f(dout[orow + c]);
  }
  __syncwarp();
  const size_t ri = ((size_t)b * nh + h) * S + i;
  const float li = lse[ri], Di = Dv[ri];
  float acc[DMAX];
#pragma unroll
  for (int c = 0; c < DMAX; ++c) acc[c] = 0.f;
  const int jend = causal ? i + 1 : S;
  for (int j = lane; j < jend; j += 32) {
    const T *kr = K + (size_t)j * ld;
    const T *vr = Vv + (size_t)j * ld;
    float sc = 0.f, dp = 0.f;
    for (int c = 0; c < d; ++c) {
      sc = fmaf(qs[wid][c], to_f(kr[c]), sc);
      dp = fmaf(dos[wid][c], to_f(vr[c]), dp);
    }
    const float ds = __expf(sc - li) * (dp - Di);
#pragma unroll
    for (int c = 0; c < DMAX; ++c)
      if (c < d) acc[c] = fmaf(ds, to_f(kr[c]), acc[c]);
  }
  T *dq = dqkv + ((size_t)b * S + i) * ld + h * d;
#pragma unroll
  for (int c = 0; c < DMAX; ++c) {
    if (c < d) {
      const float v = warp_sum(acc[c]);
      if (lane == (c % 32)) dq[c] = from_f<T>(v * scale);
    }
  }
}

template <typename T>
__global__ void attn_bwd_dkv_kernel(int S, int H, int nh, int causal, const T *__restrict__ qkv,
                                    const float *__restrict__ lse, const T *__restrict__ dout,
                                    const float *__restrict__ Dv, T *__restrict__ dqkv) {
  const int d = H / nh;
  const int lane = threadIdx.x % 32, wid = threadIdx.x / 32;
  const int j = blockIdx.x * WPB + wid;
  const int h = blockIdx.y, b = blockIdx.z;
  __shared__ float ks[WPB][DMAX], vs[WPB][DMAX];
  if (j >= S) return;
  const size_t ld = 3 * (size_t)H;
  const T *Q = qkv + ((size_t)b * S) * ld + h * d;
  const T *K = Q + H;
  const T *Vv = Q + 2 * H;
  const float scale = rsqrtf((float)d);
  for (int c = lane; c < d; c += 32) {
    ks[wid][c] = to_f(K[(size_t)j * ld + c]);
    vs[wid][c] = to_f(Vv[(size_t)j * ld + c]);
  }
  __syncwarp();
  float dk[DMAX], dv[DMAX];
#pragma unroll
  for (int c = 0; c < DMAX; ++c) dk[c] = dv[c] = 0.f;
  const int ibeg = causal ? j : 0;
  for (int i = ibeg + lane; i < S; i += 32) {
    const T *qr = Q + (size_t)i * ld;
    const T *dr = dout + ((size_t)b * S + i) * H + h * d;
    float sc = 0.f, dp = 0.f;
    for (int c = 0; c < d; ++c) {
      sc = fmaf(to_f(qr[c]) * scale, ks[wid][c], sc);
      dp = fmaf(to_f(dr[c]), vs[wid][c], dp);
    }
    const size_t ri = ((size_t)b * nh + h) * S + i;
    const float p = __expf(sc - lse[ri]);
    const float ds = p * (dp - Dv[ri]);
#pragma unroll
    for (int c = 0; c < DMAX; ++c) {
      if (c < d) {
        dv[c] = fmaf(p, to_f(dr[c]), dv[c]);
        dk[c] = fmaf(ds, to_f(qr[c]), dk[c]);
      }
    }
  }
  T *dkr = dqkv + ((size_t)b * S + j) * ld + H + h * d;
  T *dvr = dkr + H;
#pragma unroll
  for (int c = 0; c < DMAX; ++c) {
    if (c < d) {
      const float a = warp_sum(dk[c]), v = warp_sum(dv[c]);
      if (lane == (c % 32)) {
        dkr[c] = from_f<T>(a * scale);
        dvr[c] = from_f<T>(v);
      }
    }
  }
}
}  // namespace

cudaError_t attention_simt_fwd(bool bf16, int B, int S, int H, int nh, bool causal,
                               const void *qkv, void *o, float *lse, cudaStream_t s) {
  if (H / nh > DMAX) return cudaErrorInvalidValue;
  dim3 grid((S + WPB - 1) / WPB, nh, B);
  if (bf16)
    attn_fwd_kernel<__nv_bfloat16><<<grid, 32 * WPB, 0, s>>>(
        S, H, nh, causal, reinterpret_cast<const __nv_bfloat16 *>(qkv),
        reinterpret_cast<__nv_bfloat16 *>(o), lse);
  else
    attn_fwd_kernel<float><<<grid, 32 * WPB, 0, s>>>(S, H, nh, causal,
                                                     reinterpret_cast<const float *>(qkv),
                                                     reinterpret_cast<float *>(o), lse);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t attention_simt_bwd(bool bf16, int B, int S, int H, int nh, bool causal,
                               const void *qkv, const void *o, const float *lse,
                               const void *dout, void *dqkv, float *scratch, cudaStream_t s) {
  if (H / nh > DMAX) return cudaErrorInvalidValue;
  dim3 grid((S + WPB - 1) / WPB, nh, B);
#define BB_ATT_BWD(T)                                                                        \
  attn_bwd_d_kernel<T><<<grid, 32 * WPB, 0, s>>>(S, H, nh, reinterpret_cast<const T *>(o),  \
                                                 reinterpret_cast<const T *>(dout), scratch); \
  attn_bwd_dq_kernel<T><<<grid, 32 * WPB, 0, s>>>(S, H, nh, causal,                          \
      reinterpret_cast<const T *>(qkv), lse, reinterpret_cast<const T *>(dout), scratch,     \
      reinterpret_cast<T *>(dqkv));                                                          \
  attn_bwd_dkv_kernel<T><<<grid, 32 * WPB, 0, s>>>(S, H, nh, causal,                         \
      reinterpret_cast<const T *>(qkv), lse, reinterpret_cast<const T *>(dout), scratch,     \
      reinterpret_cast<T *>(dqkv));
  if (bf16) {
    BB_ATT_BWD(__nv_bfloat16)
  } else {
    BB_ATT_BWD(float)
  }
#undef BB_ATT_BWD
  g_launches += 3;
  return cudaGetLastError();
}

}  // namespace k
}  // namespace bb
