// k_common.cuh — device helpers shared by the kernels of this library.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "kernels.h"

namespace bb {
namespace k {

__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}

// GELU with the tanh approximation and its derivative.
__device__ __forceinline__ float gelu_f(float x) {
  const float c = 0.7978845608028654f;   // sqrt(2/pi)
  return 0.5f * x * (1.0f + tanhf(c * (x + 0.044715f * x * x * x)));
}
__device__ __forceinline__ float gelu_grad_f(float x) {
  const float c = 0.7978845608028654f;
  const float t = tanhf(c * (x + 0.044715f * x * x * x));
  return 0.5f * (1.0f + t) + 0.5f * x * (1.0f - t * t) * c * (1.0f + 3.0f * 0.044715f * x * x);
}

// Fast variants for bf16 outputs (tensor-core epilogues only): MUFU tanh,
// ~2^-11 relative error, below the bf16 output rounding.
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float gelu_fast(float x) {
  const float c = 0.7978845608028654f;
  return 0.5f * x * (1.0f + tanh_fast(c * (x + 0.044715f * x * x * x)));
}
__device__ __forceinline__ float gelu_grad_fast(float x) {
  const float c = 0.7978845608028654f;
  const float t = tanh_fast(c * (x + 0.044715f * x * x * x));
  return 0.5f * (1.0f + t) + 0.5f * x * (1.0f - t * t) * c * (1.0f + 3.0f * 0.044715f * x * x);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// GEMM epilogue for one output element (m, n) with fp32 accumulator `acc`.
template <typename T>
__device__ __forceinline__ void epi_store(const Gemm &g, int m, int n, float acc) {
  const size_t idx = (size_t)m * g.ldc + n;
  switch (g.epi) {
    case EPI_STORE: reinterpret_cast<T *>(g.C)[idx] = from_f<T>(acc); break;
    case EPI_BIAS:
      reinterpret_cast<T *>(g.C)[idx] = from_f<T>(acc + to_f(reinterpret_cast<const T *>(g.bias)[n]));
      break;
    case EPI_BIAS_RES:
      reinterpret_cast<T *>(g.C)[idx] =
          from_f<T>(acc + to_f(reinterpret_cast<const T *>(g.bias)[n]) +
                    to_f(reinterpret_cast<const T *>(g.res)[idx]));
      break;
    case EPI_BIAS_GELU: {
      const float pre = acc + to_f(reinterpret_cast<const T *>(g.bias)[n]);
      reinterpret_cast<T *>(g.aux)[idx] = from_f<T>(pre);
      reinterpret_cast<T *>(g.C)[idx] = from_f<T>(gelu_f(pre));
      break;
    }
    case EPI_GELU_BWD: {
      const float pre = to_f(reinterpret_cast<const T *>(g.aux)[idx]);
      reinterpret_cast<T *>(g.C)[idx] = from_f<T>(acc * gelu_grad_f(pre));
      break;
    }
    case EPI_ACC_F32: reinterpret_cast<float *>(g.C)[idx] += acc; break;
    case EPI_STORE_F32: reinterpret_cast<float *>(g.C)[idx] = acc; break;
  }
}

}  // namespace k
}  // namespace bb
