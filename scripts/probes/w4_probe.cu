// Compute-side ceilings for the batch-1 W4 decode GEMV on sm_100a (no memory):
//  1. mma.sync m16n8k16 f16->f32 dependent-chain latency (1 warp, clock64)
//  2. HMMA throughput per SM vs warps/SM (4 independent chains per warp)
//  3. LOP3 throughput per SM
//  4. the W4 inner loop itself (4 chunks = 16 lop3 x4 + 4 shf x4 + 16 HMMA in
//     two chains) from registers: weights/cycle/SM vs warps/SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o w4_probe w4_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

__device__ __forceinline__ void mma(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm volatile("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

__global__ void lat_kernel(long long* out, int n) {
  float c[4] = {};
  uint32_t a[4] = {0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u};
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) mma(c, a, 0x3c003c00u, 0x3c003c00u);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
  if (c[0] == 1.2345f) out[1] = 1;
}

__global__ void lop_kernel(uint32_t* out, int iters, uint32_t seed) {
  uint32_t v[8];
  for (int j = 0; j < 8; ++j) v[j] = seed + threadIdx.x * 7 + j;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = lop3(v[j], 0x000F000Fu, v[(j + 1) & 7]);
  uint32_t s = 0;
  for (int j = 0; j < 8; ++j) s ^= v[j];
  if (s == 0x12345678u) out[threadIdx.x] = s;
}

template <int OP>
__global__ void alu_kernel(uint32_t* out, int iters, uint32_t seed, uint32_t mul) {
  uint32_t v[8];
  for (int j = 0; j < 8; ++j) v[j] = seed + threadIdx.x * 7 + j;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (OP == 0) v[j] = __umulhi(v[j], mul) ^ j;            // IMAD.HI (+LOP3)
      if (OP == 1) v[j] = (v[j] >> (mul & 31)) + j;           // SHF (+IADD)
      if (OP == 2) v[j] = v[j] * mul + j;                     // IMAD
    }
  uint32_t s = 0;
  for (int j = 0; j < 8; ++j) s ^= v[j];
  if (s == 0x12345678u) out[threadIdx.x] = s;
}

__global__ void w4loop_kernel(float* out, int iters, uint32_t seed) {
  uint4 a4[4];
  for (int j = 0; j < 4; ++j) a4[j] = make_uint4(seed ^ j, seed * 3 + j, seed * 5 ^ j, seed + 9 * j);
  const uint32_t bx = 0x3c003c00u;
  float acc[4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int jj = 0; jj < 2; ++jj) {
      float cg[4] = {};
#pragma unroll
      for (int j = 2 * jj; j < 2 * jj + 2; ++j) {
        const uint32_t wv[4] = {a4[j].x, a4[j].y, a4[j].z, a4[j].w};
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          const uint32_t w0 = wv[2 * p], w1 = wv[2 * p + 1], w0s = w0 >> 8, w1s = w1 >> 8;
          const uint32_t lo[4] = {lop3(w0, 0x000F000Fu, 0x64006400u), lop3(w0s, 0x000F000Fu, 0x64006400u),
                                  lop3(w1, 0x000F000Fu, 0x64006400u), lop3(w1s, 0x000F000Fu, 0x64006400u)};
          const uint32_t hi[4] = {lop3(w0, 0x00F000F0u, 0x64006400u), lop3(w0s, 0x00F000F0u, 0x64006400u),
                                  lop3(w1, 0x00F000F0u, 0x64006400u), lop3(w1s, 0x00F000F0u, 0x64006400u)};
          mma(cg, lo, bx, bx);
          mma(cg, hi, bx, bx);
        }
      }
      acc[0] = fmaf(1.0f, cg[0], acc[0]);
      acc[1] = fmaf(1.0f, cg[1], acc[1]);
      acc[2] = fmaf(1.0f, cg[2], acc[2]);
      acc[3] = fmaf(1.0f, cg[3], acc[3]);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) a4[j].x += 0x11111111u;  // defeat hoisting
  }
  if (acc[0] + acc[1] + acc[2] + acc[3] == 1.2345f) out[threadIdx.x] = acc[0];
}

int main() {
  long long* dl; cudaMalloc(&dl, 64);
  float* o; cudaMalloc(&o, 1 << 16);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  lat_kernel<<<1, 32>>>(dl, 16);
  lat_kernel<<<1, 32>>>(dl, 1024);
  long long cyc; cudaMemcpy(&cyc, dl, 8, cudaMemcpyDeviceToHost);
  printf("HMMA.16816.F32 dependent latency: %.1f cycles\n", cyc / 1024.0);
  float ms;
  for (int warps : {4, 8, 16, 32}) {
    lop_kernel<<<148, warps * 32>>>((uint32_t*)o, 16, 1);
    cudaEventRecord(e0);
    lop_kernel<<<148, warps * 32>>>((uint32_t*)o, 8192, 1);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double inst = 148.0 * warps * 8192 * 8;  // warp-level lop3
    printf("LOP3 warps/SM=%2d: %.2f warp-inst/cycle/SM (at %d MHz)\n", warps, inst / 148 / (ms * 1e-3 * clk * 1e3), clk / 1000);
  }
  const char* names[3] = {"IMAD.HI+LOP3", "SHF+IADD", "IMAD"};
  for (int op = 0; op < 3; ++op) {
    auto k = op == 0 ? alu_kernel<0> : (op == 1 ? alu_kernel<1> : alu_kernel<2>);
    k<<<148, 512>>>((uint32_t*)o, 16, 1, op == 1 ? 8u : (1u << 24));
    cudaEventRecord(e0);
    k<<<148, 512>>>((uint32_t*)o, 4096, 1, op == 1 ? 8u : (1u << 24));
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double pairs = 148.0 * 16 * 4096 * 8;
    printf("%s: %.2f op-pairs/cycle/SM (warp-level)\n", names[op], pairs / 148 / (ms * 1e-3 * clk * 1e3));
  }
  for (int warps : {4, 8, 12, 16}) {
    w4loop_kernel<<<148, warps * 32>>>(o, 16, 1);
    cudaEventRecord(e0);
    w4loop_kernel<<<148, warps * 32>>>(o, 4096, 1);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double weights = 148.0 * warps * 4096 * 4096;  // 4 chunks x 1024 weights per warp-iteration
    double cyc_s = ms * 1e-3 * clk * 1e3;
    printf("W4 loop warps/SM=%2d: %.1f weights/cycle/SM  (%.0f GB/s-equivalent at 0.5 B/weight, %d MHz)\n",
           warps, weights / 148 / cyc_s, weights * 0.5 / (ms * 1e-3) / 1e9, clk / 1000);
  }
  return 0;
}
