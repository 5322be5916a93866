// Microbenchmark: peak throughput of legacy mma.sync m16n8k16 bf16 on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(float *out, int iters) {
  unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  float c[8][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0; for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float *o; cudaMalloc(&o, 148 * 8 * 1024 * 4);
  int iters = 20000;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int blocks_per_sm : {1, 2, 4}) {
    k<<<148 * blocks_per_sm, 256>>>(o, 100);
    cudaEventRecord(a);
    k<<<148 * blocks_per_sm, 256>>>(o, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double flops = 2.0 * 16 * 8 * 16 * 8.0 * iters * (148.0 * blocks_per_sm * 256 / 32);
    printf("blocks/SM %d: %.1f TFLOP/s (mma.sync bf16)\n", blocks_per_sm, flops / ms / 1e9);
  }
  return 0;
}
