// Throughput probe: legacy mma.sync m16n8k16 (f16->f32) and m16n8k32 (s8->s32)
// issued back to back with 4 independent accumulators per warp, no memory.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void hmma_loop(float* out, int iters) {
  float c[4][4] = {};
  unsigned a[4] = {0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u}, b0 = 0x3c003c00u, b1 = b0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  float s = 0; for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][3];
  if (s == 12345.f) out[threadIdx.x] = s;
}
__global__ void imma_loop(int* out, int iters) {
  int c[4][4] = {};
  unsigned a[4] = {0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u}, b0 = 0x01010101u, b1 = b0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  int s = 0; for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][3];
  if (s == 12345) out[threadIdx.x] = s;
}
int main() {
  float* o; cudaMalloc(&o, 4096);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps : {4, 8, 16, 32}) {
    const int iters = 4096;
    hmma_loop<<<148, warps * 32>>>(o, 16);
    cudaEventRecord(e0);
    hmma_loop<<<148, warps * 32>>>(o, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double n = 148.0 * warps * iters * 4;
    printf("HMMA m16n8k16 warps/SM=%2d: %.1f G mma/s = %.0f TFLOP/s\n", warps, n / ms / 1e6, n * 4096 / ms / 1e9);
    imma_loop<<<148, warps * 32>>>((int*)o, 16);
    cudaEventRecord(e0);
    imma_loop<<<148, warps * 32>>>((int*)o, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("IMMA m16n8k32 warps/SM=%2d: %.1f G mma/s = %.0f TOPS\n", warps, n / ms / 1e6, n * 8192 / ms / 1e9);
  }
  return 0;
}
