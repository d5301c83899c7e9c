// mma.sync fragment helpers for the decode GEMV (gemv.cu).
#pragma once

#include "common.cuh"

namespace msw {

__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ half2 u2h2(uint32_t u) { return *reinterpret_cast<half2*>(&u); }
__device__ __forceinline__ uint32_t h22u(half2 h) { return *reinterpret_cast<uint32_t*>(&h); }

__device__ __forceinline__ void mma_f16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                        uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_s8(int (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                       uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}


// Activations are stored permuted so that lane (g, tq) fetches both B-fragment
// registers of an MMA with one 8-byte LDS:
//   fp16, per 16-k block: [0,1,8,9 | 2,3,10,11 | 4,5,12,13 | 6,7,14,15]
//   int8, per 32-k block: [0..3,16..19 | 4..7,20..23 | 8..11,24..27 | 12..15,28..31]
__device__ __forceinline__ int perm_f16(int k) {  // pairs (k, k+1), k even, stay adjacent
  const int w = k & 15;
  return (k & ~15) + ((w & 7) >> 1) * 4 + (w >> 3) * 2 + (w & 1);
}
__device__ __forceinline__ int perm_i8(int k) {  // quads (k..k+3), k % 4 == 0, stay adjacent
  const int w = k & 31;
  return (k & ~31) + ((w & 15) >> 2) * 8 + (w >> 4) * 4 + (w & 3);
}

}  // namespace msw
