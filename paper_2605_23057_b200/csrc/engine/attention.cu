// RoPE + paged-KV append, and split-KV (flash-decoding style) attention over a
// paged cache. One kernel serves decode (1 query per sequence), continuous
// batching (ragged positions across sequences), speculative verify and
// prefill (causal: token t sees positions [0, pos[t]]): every query token is
// independent and reads its sequence's blocks through the block table, so
// prefix-cache hits (shared physical blocks) need no special casing.
//
// KV layout per layer: [block][kv_head][16 tokens][head_dim] fp16, so one
// (block, kv head) is a contiguous 16*D*2-byte run (4 KB at D=128).
#include "kernels.cuh"

namespace msw {
namespace {

__device__ __forceinline__ size_t kv_off(int slot, int hk, int Hk, int D) {
  return ((size_t(slot >> 4) * Hk + hk) * kKvBlock + (slot & 15)) * size_t(D);
}

__global__ void rope_append_kernel(const float* __restrict__ qkv, const int* __restrict__ pos,
                                   const int* __restrict__ slot, const float* __restrict__ inv_freq,
                                   int Hq, int Hk, int D, half* __restrict__ q_out,
                                   half* __restrict__ kc, half* __restrict__ vc) {
  const int t = blockIdx.x;
  const int half_d = D / 2;
  const int width = (Hq + 2 * Hk) * D;
  const float* row = qkv + size_t(t) * width;
  const float p = float(pos[t]);
  const int s = slot[t];
  for (int i = threadIdx.x; i < (Hq + Hk) * half_d; i += blockDim.x) {
    const int h = i / half_d, j = i % half_d;
    float sn, cs;
    sincosf(p * inv_freq[j], &sn, &cs);
    const float x0 = row[h * D + j], x1 = row[h * D + j + half_d];
    const float y0 = __fsub_rn(__fmul_rn(x0, cs), __fmul_rn(x1, sn));
    const float y1 = __fadd_rn(__fmul_rn(x1, cs), __fmul_rn(x0, sn));
    if (h < Hq) {
      half* q = q_out + (size_t(t) * Hq + h) * D;
      q[j] = __float2half_rn(y0);
      q[j + half_d] = __float2half_rn(y1);
    } else {
      half* k = kc + kv_off(s, h - Hq, Hk, D);
      k[j] = __float2half_rn(y0);
      k[j + half_d] = __float2half_rn(y1);
    }
  }
  for (int i = threadIdx.x; i < Hk * D; i += blockDim.x) {
    const int h = i / D, d = i % D;
    vc[kv_off(s, h, Hk, D) + d] = __float2half_rn(row[(Hq + Hk) * D + i]);
  }
}

constexpr int kAttnWarps = 4;

template <int D, int G>
__global__ void __launch_bounds__(kAttnWarps * 32)
    attention_kernel(const half* __restrict__ q, const int* __restrict__ pos,
                     const int* __restrict__ seq_of, const int* __restrict__ block_table,
                     int max_blocks, const half* __restrict__ kc, const half* __restrict__ vc, int Hq,
                     int Hk, int nsplit, float* __restrict__ part_o, float* __restrict__ part_ml,
                     float* __restrict__ o) {
  constexpr int DPL = D / 32;  // output dims per lane
  __shared__ float qs[G][D];
  __shared__ float wm[kAttnWarps][G], wl[kAttnWarps][G];
  __shared__ float wacc[kAttnWarps][G][D];
  const int t = blockIdx.x, hk = blockIdx.y, sp = blockIdx.z;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ctx = pos[t] + 1;
  const int chunk = (ctx + nsplit - 1) / nsplit;
  const int begin = sp * chunk;
  const int end = min(ctx, begin + chunk);
  const int* bt = block_table + size_t(seq_of[t]) * max_blocks;
  const float scale = 1.0f / sqrtf(float(D));

  for (int i = threadIdx.x; i < G * D; i += blockDim.x)
    qs[i / D][i % D] = __half2float(q[(size_t(t) * Hq + hk * G + i / D) * D + i % D]);
  __syncthreads();

  float m[G], l[G], acc[G][DPL];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    m[g] = -INFINITY;
    l[g] = 0.0f;
#pragma unroll
    for (int d = 0; d < DPL; ++d) acc[g][d] = 0.0f;
  }

  for (int base = begin + warp * 32; base < end; base += kAttnWarps * 32) {
    const int p = base + lane;
    float s[G];
    if (p < end) {
      const int slot = bt[p >> 4] * kKvBlock + (p & 15);
      const uint4* kr = reinterpret_cast<const uint4*>(kc + kv_off(slot, hk, Hk, D));
      float dot[G];
#pragma unroll
      for (int g = 0; g < G; ++g) dot[g] = 0.0f;
#pragma unroll 4
      for (int c = 0; c < D / 8; ++c) {
        const uint4 kv = kr[c];
        const half2* kh = reinterpret_cast<const half2*>(&kv);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 kf = __half22float2(kh[e]);
#pragma unroll
          for (int g = 0; g < G; ++g) {
            dot[g] = fmaf(qs[g][c * 8 + 2 * e], kf.x, dot[g]);
            dot[g] = fmaf(qs[g][c * 8 + 2 * e + 1], kf.y, dot[g]);
          }
        }
      }
#pragma unroll
      for (int g = 0; g < G; ++g) s[g] = dot[g] * scale;
    } else {
#pragma unroll
      for (int g = 0; g < G; ++g) s[g] = -INFINITY;
    }
    float e[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float mt = warp_max(s[g]);
      const float mn = fmaxf(m[g], mt);
      const float corr = expf(m[g] - mn);  // exp(-inf) = 0 on the first tile
      e[g] = p < end ? expf(s[g] - mn) : 0.0f;
      l[g] = l[g] * corr + warp_sum(e[g]);
      m[g] = mn;
#pragma unroll
      for (int d = 0; d < DPL; ++d) acc[g][d] *= corr;
    }
    const int n_here = min(32, end - base);
    for (int j = 0; j < n_here; ++j) {
      const int pj = base + j;
      const int slot = bt[pj >> 4] * kKvBlock + (pj & 15);
      const half* vr = vc + kv_off(slot, hk, Hk, D) + lane * DPL;
      float vf[DPL];
      if (DPL == 4) {
        const uint2 raw = *reinterpret_cast<const uint2*>(vr);
        const float2 a = __half22float2(*reinterpret_cast<const half2*>(&raw.x));
        const float2 b = __half22float2(*reinterpret_cast<const half2*>(&raw.y));
        vf[0] = a.x;
        vf[1] = a.y;
        vf[2 % DPL] = b.x;
        vf[3 % DPL] = b.y;
      } else {
#pragma unroll
        for (int d = 0; d < DPL; ++d) vf[d] = __half2float(vr[d]);
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float w = __shfl_sync(0xffffffffu, e[g], j);
#pragma unroll
        for (int d = 0; d < DPL; ++d) acc[g][d] = fmaf(w, vf[d], acc[g][d]);
      }
    }
  }

  // merge the warps of this CTA
#pragma unroll
  for (int g = 0; g < G; ++g) {
    if (lane == 0) {
      wm[warp][g] = m[g];
      wl[warp][g] = l[g];
    }
#pragma unroll
    for (int d = 0; d < DPL; ++d) wacc[warp][g][lane * DPL + d] = acc[g][d];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < G * D; i += blockDim.x) {
    const int g = i / D, d = i % D;
    float M = -INFINITY;
    for (int w = 0; w < kAttnWarps; ++w) M = fmaxf(M, wm[w][g]);
    float L = 0.0f, A = 0.0f;
    if (M != -INFINITY) {
      for (int w = 0; w < kAttnWarps; ++w) {
        const float f = expf(wm[w][g] - M);
        L += wl[w][g] * f;
        A += wacc[w][g][d] * f;
      }
    }
    const int hq = hk * G + g;
    if (nsplit == 1) {
      o[(size_t(t) * Hq + hq) * D + d] = L > 0.0f ? A / L : 0.0f;
    } else {
      const size_t idx = (size_t(t) * Hq + hq) * nsplit + sp;
      part_o[idx * D + d] = A;
      if (d == 0) {
        part_ml[idx * 2] = M;
        part_ml[idx * 2 + 1] = L;
      }
    }
  }
}

__global__ void attn_combine_kernel(const float* __restrict__ part_o,
                                    const float* __restrict__ part_ml, int Hq, int D, int nsplit,
                                    float* __restrict__ o) {
  const int t = blockIdx.x, hq = blockIdx.y;
  const size_t base = (size_t(t) * Hq + hq) * nsplit;
  float M = -INFINITY;
  for (int s = 0; s < nsplit; ++s) M = fmaxf(M, part_ml[(base + s) * 2]);
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    float L = 0.0f, A = 0.0f;
    for (int s = 0; s < nsplit; ++s) {
      const float ms = part_ml[(base + s) * 2];
      if (ms == -INFINITY) continue;
      const float f = expf(ms - M);
      L += part_ml[(base + s) * 2 + 1] * f;
      A += part_o[(base + s) * D + d] * f;
    }
    o[(size_t(t) * Hq + hq) * D + d] = L > 0.0f ? A / L : 0.0f;
  }
}

template <int D>
void attn_d(int G, dim3 grid, const half* q, const int* pos, const int* seq_of, const int* bt,
            int maxb, const half* kc, const half* vc, int Hq, int Hk, int nsplit, float* po,
            float* pml, float* o, cudaStream_t st) {
  const int thr = kAttnWarps * 32;
#define MSW_ATT(GG)                                                                          \
  case GG:                                                                                   \
    attention_kernel<D, GG><<<grid, thr, 0, st>>>(q, pos, seq_of, bt, maxb, kc, vc, Hq, Hk, \
                                                  nsplit, po, pml, o);                       \
    break;
  switch (G) {
    MSW_ATT(1)
    MSW_ATT(2)
    MSW_ATT(4)
    MSW_ATT(8)
    default: throw ConfigErr("attention: GQA group must be 1, 2, 4 or 8");
  }
#undef MSW_ATT
}

}  // namespace

void launch_rope_append(const float* qkv, int T, const int* pos, const int* slot,
                        const float* inv_freq, const AttnShape& a, half* q_out, half* kc, half* vc,
                        cudaStream_t st) {
  rope_append_kernel<<<T, 256, 0, st>>>(qkv, pos, slot, inv_freq, a.n_heads, a.n_kv_heads,
                                        a.head_dim, q_out, kc, vc);
  MSW_LAUNCH_CHECK();
}

void launch_attention(const half* q, int T, const int* pos, const int* seq_of,
                      const int* block_table, const half* kc, const half* vc, const AttnShape& a,
                      int nsplit, float* part_o, float* part_ml, float* o, cudaStream_t st) {
  const int G = a.n_heads / a.n_kv_heads;
  const dim3 grid(T, a.n_kv_heads, nsplit);
  if (a.head_dim == 128)
    attn_d<128>(G, grid, q, pos, seq_of, block_table, a.max_blocks_per_seq, kc, vc, a.n_heads,
                a.n_kv_heads, nsplit, part_o, part_ml, o, st);
  else if (a.head_dim == 64)
    attn_d<64>(G, grid, q, pos, seq_of, block_table, a.max_blocks_per_seq, kc, vc, a.n_heads,
               a.n_kv_heads, nsplit, part_o, part_ml, o, st);
  else
    throw ConfigErr("attention: head_dim must be 64 or 128");
  MSW_LAUNCH_CHECK();
  if (nsplit > 1) {
    attn_combine_kernel<<<dim3(T, a.n_heads), 128, 0, st>>>(part_o, part_ml, a.n_heads,
                                                           a.head_dim, nsplit, o);
    MSW_LAUNCH_CHECK();
  }
}

}  // namespace msw
