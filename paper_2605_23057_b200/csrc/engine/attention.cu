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
#include "mma_frag.cuh"

namespace msw {
#ifdef MSW_TRACE
__device__ unsigned long long* g_attn_trace = nullptr;
extern "C" int msw_attn_trace_set(void* buf) {
  return cudaMemcpyToSymbol(g_attn_trace, &buf, sizeof(buf)) == cudaSuccess ? 0 : 1;
}
// globaltimer at event e of CTA (blockIdx linearised): buf[cta * 8 + e]
#define ATT_TP(e)                                                                           \
  do {                                                                                      \
    if (g_attn_trace && threadIdx.x == 0) {                                                 \
      unsigned long long g_;                                                                \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_));                                \
      const int c_ = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;        \
      g_attn_trace[c_ * 8 + (e)] = g_;                                                      \
    }                                                                                       \
  } while (0)
#else
#define ATT_TP(e) \
  do {            \
  } while (0)
#endif
namespace {

__device__ __forceinline__ size_t kv_off(int slot, int hk, int Hk, int D) {
  return ((size_t(slot >> 4) * Hk + hk) * kKvBlock + (slot & 15)) * size_t(D);
}

// KV-cache compression (MSW_MODE_KV_COMPRESSION): K / V stored as FP8 E4M3,
// one byte per element in the same [block][kv_head][16][D] layout.
// fp16 pair -> e4m3 pair (round to nearest even, saturating to +-448), element
// 2i in the low byte; and back (exact: e4m3 is a subset of fp16).
__device__ __forceinline__ uint16_t h2_to_e4m3x2(half lo, half hi) {
  uint16_t r;
  const uint32_t v = uint32_t(__half_as_ushort(lo)) | (uint32_t(__half_as_ushort(hi)) << 16);
  asm("cvt.rn.satfinite.e4m3x2.f16x2 %0, %1;" : "=h"(r) : "r"(v));
  return r;
}
__device__ __forceinline__ uint32_t e4m3x2_to_h2(uint16_t v) {
  uint32_t r;
  asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(r) : "h"(v));
  return r;
}

__global__ void rope_table_kernel(const float* __restrict__ inv_freq, int half_d, int max_pos,
                                  float2* __restrict__ table) {
  const int total = max_pos * half_d;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int p = i / half_d, j = i % half_d;
    float sn, cs;
    sincosf(float(p) * inv_freq[j], &sn, &cs);  // fp32 angle, as the oracle
    table[i] = make_float2(cs, sn);
  }
}

__global__ void rope_append_kernel(const float* __restrict__ qkv, const int* __restrict__ pos,
                                   const int* __restrict__ slot, const float2* __restrict__ rope,
                                   int Hq, int Hk, int D, half* __restrict__ q_out,
                                   half* __restrict__ kc, half* __restrict__ vc) {
  pdl_wait();
  pdl_trigger();
  const int t = blockIdx.x;
  const int half_d = D / 2;
  const int width = (Hq + 2 * Hk) * D;
  const float* row = qkv + size_t(t) * width;
  const int pi = pos[t];
  const int s = slot[t];
  for (int i = threadIdx.x; i < (Hq + Hk) * half_d; i += blockDim.x) {
    const int h = i / half_d, j = i % half_d;
    const float2 r = rope[size_t(pi) * half_d + j];
    const float cs = r.x, sn = r.y;
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

// Positions per split: at least kMinChunk so short contexts use few CTAs.
constexpr int kMinChunk = 64;
__device__ __forceinline__ int split_chunk(int ctx, int nsplit) {
  const int c = (ctx + nsplit - 1) / nsplit;
  return ((max(c, kMinChunk) + 31) / 32) * 32;
}

// FUSED (decode / continuous batching: every query token is the newest token
// of its own sequence): RoPE of q and of the new k happens here from the
// fp32 qkv row; the split-0 CTA appends k/v to the paged cache, and every CTA
// uses the fresh k/v from shared memory for the query's own position instead
// of reading the cache (no cross-CTA ordering needed).
constexpr int kKvPad = 8;  // halves of padding per staged K/V row (bank-conflict free LDS.128)

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

template <int D, int G, bool FUSED>
__global__ void __launch_bounds__(kAttnWarps * 32)
    attention_kernel(const half* __restrict__ q, const float* __restrict__ qkv,
                     const float* __restrict__ inv_freq, const int* __restrict__ pos,
                     const int* __restrict__ slot, const int* __restrict__ seq_of,
                     const int* __restrict__ block_table, int max_blocks, half* __restrict__ kc,
                     half* __restrict__ vc, int Hq, int Hk, int nsplit,
                     float* __restrict__ part_o, float* __restrict__ part_ml,
                     float* __restrict__ o) {
  constexpr int DPL = D / 32;  // output dims per lane
  __shared__ float qs[G][D];
  __shared__ float knew[D], vnew[D];
  __shared__ float wm[kAttnWarps][G], wl[kAttnWarps][G];
  __shared__ float wacc[kAttnWarps][G][D];
  const int t = blockIdx.x, hk = blockIdx.y, sp = blockIdx.z;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  pdl_wait();
  pdl_trigger();
  const int p_self = pos[t];
  const int ctx = p_self + 1;
  const int chunk = split_chunk(ctx, nsplit);
  const int begin = sp * chunk;
  if (begin >= ctx) return;  // inactive split (combine ignores it)
  const bool single = chunk >= ctx;
  const int end = min(ctx, begin + chunk);
  const int* bt = block_table + size_t(seq_of[t]) * max_blocks;
  const float scale = 1.0f / sqrtf(float(D));

  if (FUSED) {
    const int width = (Hq + 2 * Hk) * D;
    const float* row = qkv + size_t(t) * width;
    const float pf = float(p_self);
    for (int i = threadIdx.x; i < (G + 1) * (D / 2); i += blockDim.x) {
      const int h = i / (D / 2), j = i % (D / 2);
      const float* src = h < G ? row + size_t(hk * G + h) * D : row + size_t(Hq + hk) * D;
      float sn, cs;
      sincosf(pf * inv_freq[j], &sn, &cs);
      const float x0 = src[j], x1 = src[j + D / 2];
      const float y0 = __half2float(__float2half_rn(__fsub_rn(__fmul_rn(x0, cs), __fmul_rn(x1, sn))));
      const float y1 = __half2float(__float2half_rn(__fadd_rn(__fmul_rn(x1, cs), __fmul_rn(x0, sn))));
      if (h < G) {
        qs[h][j] = y0;
        qs[h][j + D / 2] = y1;
      } else {
        knew[j] = y0;
        knew[j + D / 2] = y1;
      }
    }
    for (int d = threadIdx.x; d < D; d += blockDim.x)
      vnew[d] = __half2float(__float2half_rn(row[size_t(Hq + Hk + hk) * D + d]));
    __syncthreads();
    if (sp == 0) {
      const size_t off = kv_off(slot[t], hk, Hk, D);
      for (int d = threadIdx.x; d < D; d += blockDim.x) {
        kc[off + d] = __float2half_rn(knew[d]);
        vc[off + d] = __float2half_rn(vnew[d]);
      }
    }
  } else {
    for (int i = threadIdx.x; i < G * D; i += blockDim.x)
      qs[i / D][i % D] = __half2float(q[(size_t(t) * Hq + hk * G + i / D) * D + i % D]);
  }
  __syncthreads();

  float m[G], l[G], acc[G][DPL];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    m[g] = -INFINITY;
    l[g] = 0.0f;
#pragma unroll
    for (int d = 0; d < DPL; ++d) acc[g][d] = 0.0f;
  }

  // per-warp K tile in shared memory, staged with coalesced 16-byte pieces
  // (2 rows per warp instruction for D = 128) instead of lane = position loads
  constexpr int RS = D + kKvPad, CPR = D / 8, RPI = 32 / CPR;
  extern __shared__ __align__(16) half ks_smem[];
  half* sK = ks_smem + size_t(warp) * 32 * RS;
  for (int base = begin + warp * 32; base < end; base += kAttnWarps * 32) {
    __syncwarp();  // the previous tile's rows are consumed
#pragma unroll 4
    for (int i = 0; i < 32 / RPI; ++i) {
      const int r = i * RPI + lane / CPR;
      const int pr = base + r;
      if (pr < end && !(FUSED && pr == p_self)) {
        const int sl = bt[pr >> 4] * kKvBlock + (pr & 15);
        cp_async16(sK + r * RS + (lane % CPR) * 8, kc + kv_off(sl, hk, Hk, D) + (lane % CPR) * 8);
      }
    }
    cp_async_wait_all();
    __syncwarp();
    const int p = base + lane;
    float s[G];
    if (p < end) {
      float dot[G];
#pragma unroll
      for (int g = 0; g < G; ++g) dot[g] = 0.0f;
      if (FUSED && p == p_self) {
        for (int d = 0; d < D; ++d) {
#pragma unroll
          for (int g = 0; g < G; ++g) dot[g] = fmaf(qs[g][d], knew[d], dot[g]);
        }
      } else {
        const uint4* kr = reinterpret_cast<const uint4*>(sK + lane * RS);
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
    for (int j0 = 0; j0 < n_here; j0 += 8) {
      float vf[8][DPL];
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {  // issue up to 8 row loads before consuming any
        const int pj = base + j0 + jj;
        if (j0 + jj >= n_here) {
#pragma unroll
          for (int d = 0; d < DPL; ++d) vf[jj][d] = 0.0f;
        } else if (FUSED && pj == p_self) {
#pragma unroll
          for (int d = 0; d < DPL; ++d) vf[jj][d] = vnew[lane * DPL + d];
        } else {
          const int sl = bt[pj >> 4] * kKvBlock + (pj & 15);
          const half* vr = vc + kv_off(sl, hk, Hk, D) + lane * DPL;
#pragma unroll
          for (int d = 0; d < DPL; d += 2) {
            const float2 f = __half22float2(*reinterpret_cast<const half2*>(vr + d));
            vf[jj][d] = f.x;
            vf[jj][d + 1] = f.y;
          }
        }
      }
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const float w = __shfl_sync(0xffffffffu, e[g], (j0 + jj) & 31);
#pragma unroll
          for (int d = 0; d < DPL; ++d) acc[g][d] = fmaf(w, vf[jj][d], acc[g][d]);
        }
      }
    }
  }

  ATT_TP(3);
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
    if (single) {
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

// Decode kernel geometry: 8 warps x 32 positions per CTA and >= 256 positions
// per split, so a context of up to 256 positions is one CTA per kv head with
// one tile per warp and no cross-CTA merge. (Measured in-graph, 8B W4, ctx 202:
// the 4-warp / 64-position version spent 6.5 of its 17.8 us per layer in the
// fence + atomic + last-CTA split merge; scripts/attn_timeline.py.)
constexpr int kRunMax = 6;  // = kGemvMaxTokens: longest run of one sequence in one launch
#ifndef MSW_ATTN_MMA
#define MSW_ATTN_MMA 1  // decode attention tile on mma.sync (0: scalar FMA loops)
#endif
constexpr int kDecMinChunk = 256;
__device__ __forceinline__ int split_chunk_dec(int ctx, int nsplit) {
  const int c = (ctx + nsplit - 1) / nsplit;
  return ((max(c, kDecMinChunk) + 31) / 32) * 32;
}

// Decode / continuous-batching attention (each query token is the newest
// token of its own sequence). Per CTA: one (token, kv head, split).
//  * before griddepcontrol.wait: the K rows and V slices of the first tile of
//    this split's range are loaded (positions < pos[t] are immutable history;
//    pos / slot / block table were written by kernels that completed before
//    the previous one), so the cache reads overlap the QKV GEMV's tail;
//  * after the wait: RoPE of q and the new k from the fp32 qkv row; the
//    split-0 CTA appends k / v to the paged cache; the query's own position
//    uses the fresh k / v from shared memory;
//  * splits are merged in-kernel: every split writes (m, l, acc) partials and
//    the last CTA to finish (atomic counter) combines them, so there is no
//    separate combine launch.

// KV8: the paged cache holds FP8 E4M3 (KV-cache compression mode): history
// rows are widened to fp16 while staged, and this launch's new keys / values
// are rounded through E4M3 before use and stored as E4M3, so every position
// the query attends to carries the cache's precision.
// PT = positions per warp tile (32; 16 is supported for an fp16 cache).
template <int D, int G, int W, bool KV8, int PT>
__global__ void __launch_bounds__(W * 32)
    attn_decode_kernel(const float* __restrict__ qkv, const float2* __restrict__ rope,
                       const int* __restrict__ pos, const int* __restrict__ slot,
                       const int* __restrict__ seq_of, const int* __restrict__ block_table,
                       int max_blocks, typename std::conditional<KV8, uint8_t, half>::type* __restrict__ kc,
                       typename std::conditional<KV8, uint8_t, half>::type* __restrict__ vc, int Hq, int Hk,
                       int nsplit, float* __restrict__ part_o, float* __restrict__ part_ml,
                       int* __restrict__ counters, float* __restrict__ o, int run) {
  constexpr int DPL = D / 32;
  constexpr int RS = D + kKvPad;  // staged row stride (halves)
  static_assert(PT == 32 || (PT == 16 && !KV8), "warp tile: 32 positions, or 16 (fp16 cache)");
  constexpr int NTL = PT / 8;    // QK n-tiles of 8 positions
  constexpr int KSV = PT / 16;   // PV k-steps of 16 positions
  extern __shared__ __align__(16) half kv_smem[];  // [warp][K|V][PT][RS]
  __shared__ __align__(16) float qs[G][D];
  // new keys / values of this launch: row 0 only for independent tokens; rows
  // 0..t for a run (tokens 0..T-1 = consecutive positions of one sequence)
  __shared__ __align__(16) half knew_all[kRunMax][D], vnew_all[kRunMax][D];
  half* const knew = knew_all[0];
  half* const vnew = vnew_all[0];
  __shared__ float wm[W][G], wl[W][G];
  __shared__ __align__(16) float wacc[W][G][D];
  __shared__ int is_last;
  const int t = blockIdx.x, hk = blockIdx.y, sp = blockIdx.z;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  ATT_TP(0);
  const int p_self = pos[t];
  const int ctx = p_self + 1;
  // positions [p_new, p_self] come from this launch's qkv rows, not the cache:
  // the own position for independent tokens; every earlier token of the run
  // too (their cache rows are appended by other CTAs of this launch)
  const int p_new = run ? p_self - t : p_self;
  const int chunk = split_chunk_dec(ctx, nsplit);
  const int begin = sp * chunk;
  if (begin >= ctx) {
    pdl_wait();
    pdl_trigger();
    ATT_TP(7);  // idle split
    return;
  }
  const int end = min(ctx, begin + chunk);
  const int active = (ctx + chunk - 1) / chunk;
  const int* bt = block_table + size_t(seq_of[t]) * max_blocks;
  half* sK = kv_smem + size_t(warp) * 2 * PT * RS;
  half* sV = sK + PT * RS;

  // stage one PT-position tile of cached K / V rows. Lanes cover consecutive
  // 16-byte pieces of the same row (32 / (D/8) rows per instruction), so one
  // warp instruction touches 2 (D = 128) contiguous rows instead of 32
  // scattered ones: 8x fewer L1 wavefronts than lane = position.
  constexpr int CPR = D / 8, RPI = 32 / CPR;
  auto stage_tile = [&](int base) {
    const int c = lane % CPR;
#pragma unroll 4
    for (int i = 0; i < PT / RPI; ++i) {
      const int r = i * RPI + lane / CPR;
      const int p = base + r;
      if (p < end && p < p_new) {
        const int sl = bt[p >> 4] * kKvBlock + (p & 15);
        cp_async16(sK + r * RS + c * 8, kc + kv_off(sl, hk, Hk, D) + c * 8);
        cp_async16(sV + r * RS + c * 8, vc + kv_off(sl, hk, Hk, D) + c * 8);
      }
    }
  };
  // KV8: the tile's E4M3 rows are copied asynchronously, raw, into the top
  // kRaw8 bytes of each staged row (D bytes ending at the padded row end),
  // then widened in place by widen_tile: lane = row, the row's raw bytes are
  // all read into registers before any fp16 store, so the overlap of the
  // fp16 region [0, 2D) with the raw one [2 RS - D, 2 RS) is harmless.
  constexpr int kRaw8 = 2 * RS - D;  // byte offset of the raw row (multiple of 16)
  constexpr int CPR8 = D / 16, RPI8 = 32 / CPR8;
  auto stage_tile8 = [&](int base) {
    const int c = lane % CPR8;
#pragma unroll 4
    for (int i = 0; i < 32 / RPI8; ++i) {
      const int r = i * RPI8 + lane / CPR8;
      const int p = base + r;
      if (p < end && p < p_new) {
        const int sl = bt[p >> 4] * kKvBlock + (p & 15);
        cp_async16(reinterpret_cast<uint8_t*>(sK + r * RS) + kRaw8 + c * 16,
                   kc + kv_off(sl, hk, Hk, D) + c * 16);
        cp_async16(reinterpret_cast<uint8_t*>(sV + r * RS) + kRaw8 + c * 16,
                   vc + kv_off(sl, hk, Hk, D) + c * 16);
      }
    }
  };
  auto widen_tile = [&]() {
#pragma unroll
    for (int kv = 0; kv < 2; ++kv) {
      half* row = (kv == 0 ? sK : sV) + lane * RS;
      uint4 raw[CPR8];
#pragma unroll
      for (int c = 0; c < CPR8; ++c)
        raw[c] = *reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(row) + kRaw8 + c * 16);
#pragma unroll
      for (int c = 0; c < CPR8; ++c) {
        const uint32_t w[4] = {raw[c].x, raw[c].y, raw[c].z, raw[c].w};
        uint4 lo, hi;
        lo.x = e4m3x2_to_h2(uint16_t(w[0]));
        lo.y = e4m3x2_to_h2(uint16_t(w[0] >> 16));
        lo.z = e4m3x2_to_h2(uint16_t(w[1]));
        lo.w = e4m3x2_to_h2(uint16_t(w[1] >> 16));
        hi.x = e4m3x2_to_h2(uint16_t(w[2]));
        hi.y = e4m3x2_to_h2(uint16_t(w[2] >> 16));
        hi.z = e4m3x2_to_h2(uint16_t(w[3]));
        hi.w = e4m3x2_to_h2(uint16_t(w[3] >> 16));
        *reinterpret_cast<uint4*>(row + c * 16) = lo;
        *reinterpret_cast<uint4*>(row + c * 16 + 8) = hi;
      }
    }
  };
  const int first = begin + warp * PT;
  if (first < end) {  // cache history only: safe before the wait
    if constexpr (KV8) stage_tile8(first);
    else stage_tile(first);
  }
  // the RoPE row of this position is a cold table row: fetch it before the wait
  // too (pos was written by the previous step's advance, long complete).
  // Items after the wait: (G + 1) * D / 2 RoPE pairs (q heads, new key), then
  // D value elements, all loaded in one round trip.
  constexpr int kRopeItems = (G + 1) * (D / 2), kItems = kRopeItems + D;
  constexpr int kIt = (kItems + W * 32 - 1) / (W * 32);
  const float2* rp = rope + size_t(p_self) * (D / 2);
  float2 rr[kIt];
#pragma unroll
  for (int it = 0; it < kIt; ++it) {
    const int i = threadIdx.x + it * W * 32;
    if (i < kRopeItems) rr[it] = rp[i % (D / 2)];
  }

  // the append slot too (a dependent global load after the wait cost ~0.8 us)
  const int slot_t = sp == 0 ? slot[t] : 0;

  pdl_wait();
  ATT_TP(1);
  pdl_trigger();
  {  // RoPE of this kv head's G query heads and the new key (table lookup)
    const float* row = qkv + size_t(t) * (Hq + 2 * Hk) * D;
    float xa[kIt], xb[kIt];
#pragma unroll
    for (int it = 0; it < kIt; ++it) {
      const int i = threadIdx.x + it * W * 32;
      if (i < kRopeItems) {
        const int h = i / (D / 2), j = i % (D / 2);
        const float* src = h < G ? row + size_t(hk * G + h) * D : row + size_t(Hq + hk) * D;
        xa[it] = src[j];
        xb[it] = src[j + D / 2];
      } else if (i < kItems) {
        xa[it] = row[size_t(Hq + Hk + hk) * D + (i - kRopeItems)];
      }
    }
#pragma unroll
    for (int it = 0; it < kIt; ++it) {
      const int i = threadIdx.x + it * W * 32;
      if (i < kRopeItems) {
        const int h = i / (D / 2), j = i % (D / 2);
        const float2 r = rr[it];
        const float x0 = xa[it], x1 = xb[it];
        const half y0 = __float2half_rn(__fsub_rn(__fmul_rn(x0, r.x), __fmul_rn(x1, r.y)));
        const half y1 = __float2half_rn(__fadd_rn(__fmul_rn(x1, r.x), __fmul_rn(x0, r.y)));
        if (h < G) {
          qs[h][j] = __half2float(y0);
          qs[h][j + D / 2] = __half2float(y1);
        } else {
          knew[j] = y0;
          knew[j + D / 2] = y1;
        }
      } else if (i < kItems) {
        vnew[i - kRopeItems] = __float2half_rn(xa[it]);
      }
    }
  }
  if (run && t > 0) {  // keys / values of the run's earlier tokens (rows 0..t-1)
    for (int i = threadIdx.x; i < t * (D / 2); i += blockDim.x) {
      const int q = 1 + i / (D / 2), j = i % (D / 2);  // row q: token t - q at p_self - q
      const float* rw = qkv + size_t(t - q) * (Hq + 2 * Hk) * D;
      const float2 rt = rope[size_t(p_self - q) * (D / 2) + j];
      const float* src = rw + size_t(Hq + hk) * D;
      const float x0 = src[j], x1 = src[j + D / 2];
      knew_all[q][j] = __float2half_rn(__fsub_rn(__fmul_rn(x0, rt.x), __fmul_rn(x1, rt.y)));
      knew_all[q][j + D / 2] = __float2half_rn(__fadd_rn(__fmul_rn(x1, rt.x), __fmul_rn(x0, rt.y)));
    }
    for (int i = threadIdx.x; i < t * D; i += blockDim.x) {
      const int q = 1 + i / D, d = i % D;
      vnew_all[q][d] = __float2half_rn(qkv[size_t(t - q) * (Hq + 2 * Hk) * D + size_t(Hq + Hk + hk) * D + d]);
    }
  }
  __syncthreads();
  if constexpr (KV8) {  // the new rows at the cache's precision (E4M3 round trip)
    const int rows = run ? t + 1 : 1;
    for (int i = threadIdx.x; i < rows * (D / 2); i += blockDim.x) {
      const int q = i / (D / 2), d = 2 * (i % (D / 2));
      const uint32_t kk = e4m3x2_to_h2(h2_to_e4m3x2(knew_all[q][d], knew_all[q][d + 1]));
      const uint32_t vv = e4m3x2_to_h2(h2_to_e4m3x2(vnew_all[q][d], vnew_all[q][d + 1]));
      *reinterpret_cast<uint32_t*>(&knew_all[q][d]) = kk;
      *reinterpret_cast<uint32_t*>(&vnew_all[q][d]) = vv;
    }
    __syncthreads();
  }
  ATT_TP(2);
  if (sp == 0) {
    const size_t off = kv_off(slot_t, hk, Hk, D);
    if constexpr (KV8) {
      for (int d = 2 * threadIdx.x; d < D; d += 2 * blockDim.x) {
        *reinterpret_cast<uint16_t*>(kc + off + d) = h2_to_e4m3x2(knew[d], knew[d + 1]);
        *reinterpret_cast<uint16_t*>(vc + off + d) = h2_to_e4m3x2(vnew[d], vnew[d + 1]);
      }
    } else {
      for (int d = threadIdx.x; d < D; d += blockDim.x) {
        kc[off + d] = knew[d];
        vc[off + d] = vnew[d];
      }
    }
  }
  const float scale = rsqrtf(float(D));
#if MSW_ATTN_MMA
  // Tensor-pipe tile (mma.sync m16n8k16, fp32 accumulate): rows = the G query
  // heads (16-row A tile, rows >= G zero), QK over 4 n-tiles of 8 positions,
  // P (fp16, FA2 register reuse) x V with V fragments from ldmatrix.trans.
  constexpr int KS = D / 16, DT = D / 8;
  const int g = lane >> 2, tq = lane & 3;
  uint32_t qa[KS][2];
#pragma unroll
  for (int kk = 0; kk < KS; ++kk) {
    const int k0 = kk * 16 + 2 * tq;
    qa[kk][0] = g < G ? h22u(__floats2half2_rn(qs[g < G ? g : 0][k0], qs[g < G ? g : 0][k0 + 1])) : 0u;
    qa[kk][1] = g < G ? h22u(__floats2half2_rn(qs[g < G ? g : 0][k0 + 8], qs[g < G ? g : 0][k0 + 9])) : 0u;
  }
  float mrow = -INFINITY, lrow = 0.0f;
  float acc[DT][4];
#pragma unroll
  for (int dt = 0; dt < DT; ++dt) acc[dt][0] = acc[dt][1] = acc[dt][2] = acc[dt][3] = 0.0f;
#pragma unroll 1
  for (int base = first; base < end; base += W * PT) {
    if (base != first) {
      __syncwarp();
      if constexpr (KV8) stage_tile8(base);
      else stage_tile(base);
    }
    cp_async_wait_all();
    if constexpr (KV8) {
      __syncwarp();  // every lane's raw rows landed
      widen_tile();
      __syncwarp();
    }
    if (base == first) ATT_TP(6);  // warp 0: first tile staged
    {
      // this launch's new rows [p_new, p_self] come from smem, not the cache;
      // V rows past `end` are zeroed (P = 0 there, but 0 x stale-NaN V would
      // poison the MMA). The whole warp copies, one 16-byte piece per lane.
      constexpr int PPR = D / 8;  // 16-byte pieces per row
      const int r0 = max(base, p_new) - base, r1 = min(base + PT, min(p_self + 1, end)) - base;
      for (int i = lane; i < max(0, r1 - r0) * 2 * PPR; i += 32) {
        const int r = r0 + i / (2 * PPR), c = i % (2 * PPR);
        const int q = p_self - (base + r);
        const half* src = c < PPR ? knew_all[q] + c * 8 : vnew_all[q] + (c - PPR) * 8;
        half* dst = (c < PPR ? sK + c * 8 : sV + (c - PPR) * 8) + r * RS;
        *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src);
      }
      const int z0 = max(0, end - base);
      for (int i = lane; i < max(0, PT - z0) * PPR; i += 32)
        *reinterpret_cast<uint4*>(sV + (z0 + i / PPR) * RS + (i % PPR) * 8) = make_uint4(0u, 0u, 0u, 0u);
    }
    __syncwarp();
    float sc[NTL][2];
#pragma unroll
    for (int nt = 0; nt < NTL; ++nt) {
      float c4[4] = {0.f, 0.f, 0.f, 0.f};
      // B fragments of two k-steps per ldmatrix.x4 (K rows = positions, non-trans)
      const half* kr = sK + (nt * 8 + (lane & 7)) * RS + (lane >> 3) * 8;
#pragma unroll
      for (int kk = 0; kk < KS; kk += 2) {
        uint32_t b[4];
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                     : "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3])
                     : "r"(smem_u32(kr + kk * 16)));
        const uint32_t a0[4] = {qa[kk][0], 0u, qa[kk][1], 0u};
        mma_f16(c4, a0, b[0], b[1]);
        const uint32_t a1[4] = {qa[kk + 1][0], 0u, qa[kk + 1][1], 0u};
        mma_f16(c4, a1, b[2], b[3]);
      }
#pragma unroll
      for (int e2 = 0; e2 < 2; ++e2) {
        const int pp = base + nt * 8 + 2 * tq + e2;
        sc[nt][e2] = pp < end ? c4[e2] * scale : -INFINITY;
      }
    }
    float mt = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < NTL; ++nt) mt = fmaxf(mt, fmaxf(sc[nt][0], sc[nt][1]));
    mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, 1));
    mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, 2));
    const float mn = fmaxf(mrow, mt);
    const float corr = __expf(mrow - mn);
    float ls = 0.0f;
    uint32_t pa[KSV][2];
#pragma unroll
    for (int nt = 0; nt < NTL; ++nt) {
      const float e0 = sc[nt][0] == -INFINITY ? 0.0f : __expf(sc[nt][0] - mn);
      const float e1 = sc[nt][1] == -INFINITY ? 0.0f : __expf(sc[nt][1] - mn);
      ls += e0 + e1;
      pa[nt >> 1][nt & 1] = h22u(__floats2half2_rn(e0, e1));
    }
    ls += __shfl_xor_sync(0xffffffffu, ls, 1);
    ls += __shfl_xor_sync(0xffffffffu, ls, 2);
    lrow = lrow * corr + ls;
    mrow = mn;
#pragma unroll
    for (int dt = 0; dt < DT; ++dt) {
      acc[dt][0] *= corr;
      acc[dt][1] *= corr;
    }
    const int n_here = min(PT, end - base);
    if (base == first && active == 1) ATT_TP(5);  // warp 0: QK + softmax done (single split)
#pragma unroll
    for (int ks = 0; ks < KSV; ++ks) {
      if (ks * 16 >= n_here) break;  // warp-uniform
      const uint32_t a4[4] = {g < G ? pa[ks][0] : 0u, 0u, g < G ? pa[ks][1] : 0u, 0u};
      const half* vrow = sV + (ks * 16 + (lane & 15)) * RS;
#pragma unroll
      for (int dt = 0; dt < DT; ++dt) {
        uint32_t b0, b1;
        asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0, %1}, [%2];"
                     : "=r"(b0), "=r"(b1)
                     : "r"(smem_u32(vrow + dt * 8)));
        mma_f16(acc[dt], a4, b0, b1);
      }
    }
  }
  // per-warp (m, l, acc) -> shared, rows g < G held by the tq lanes
  if (g < G) {
    if (tq == 0) {
      wm[warp][g < G ? g : 0] = mrow;
      wl[warp][g < G ? g : 0] = lrow;
    }
#pragma unroll
    for (int dt = 0; dt < DT; ++dt) {
      wacc[warp][g < G ? g : 0][dt * 8 + 2 * tq] = acc[dt][0];
      wacc[warp][g < G ? g : 0][dt * 8 + 2 * tq + 1] = acc[dt][1];
    }
  }
#else
  static_assert(PT == 32, "scalar decode attention: 32-position warp tiles");
  const float scale = rsqrtf(float(D));
  float m[G], l[G], acc[G][DPL];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    m[g] = -INFINITY;
    l[g] = 0.0f;
#pragma unroll
    for (int d = 0; d < DPL; ++d) acc[g][d] = 0.0f;
  }
#pragma unroll 1
  for (int base = first; base < end; base += W * 32) {
    if (base != first) {
      __syncwarp();
      stage_tile(base);
    }
    cp_async_wait_all();
    const int p = base + lane;
    if (p >= p_new && p <= p_self) {  // this launch's new rows come from smem, not the cache
      const half* kn = knew_all[p_self - p];
      const half* vn = vnew_all[p_self - p];
#pragma unroll 1
      for (int c = 0; c < D / 8; ++c) {
        *reinterpret_cast<uint4*>(sK + lane * RS + c * 8) = *reinterpret_cast<const uint4*>(kn + c * 8);
        *reinterpret_cast<uint4*>(sV + lane * RS + c * 8) = *reinterpret_cast<const uint4*>(vn + c * 8);
      }
    }
    __syncwarp();
    float s[G];
#pragma unroll
    for (int g = 0; g < G; ++g) s[g] = 0.0f;
    if (p < end) {
      const half* kr = sK + lane * RS;
#pragma unroll  // 8 warps x 256 threads: registers allow full ILP over D
      for (int c = 0; c < D / 8; ++c) {
        const uint4 kv = *reinterpret_cast<const uint4*>(kr + c * 8);
        const half2* kh = reinterpret_cast<const half2*>(&kv);
        const float2 k0 = __half22float2(kh[0]), k1 = __half22float2(kh[1]);
        const float2 k2 = __half22float2(kh[2]), k3 = __half22float2(kh[3]);
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const float4 q0 = *reinterpret_cast<const float4*>(&qs[g][c * 8]);
          const float4 q1 = *reinterpret_cast<const float4*>(&qs[g][c * 8 + 4]);
          s[g] = fmaf(q0.x, k0.x, fmaf(q0.y, k0.y, fmaf(q0.z, k1.x, fmaf(q0.w, k1.y, s[g]))));
          s[g] = fmaf(q1.x, k2.x, fmaf(q1.y, k2.y, fmaf(q1.z, k3.x, fmaf(q1.w, k3.y, s[g]))));
        }
      }
    }
    float e[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float sv = p < end ? s[g] * scale : -INFINITY;
      const float mn = fmaxf(m[g], warp_max(sv));
      const float corr = __expf(m[g] - mn);
      e[g] = p < end ? __expf(sv - mn) : 0.0f;
      l[g] = l[g] * corr + warp_sum(e[g]);
      m[g] = mn;
#pragma unroll
      for (int d = 0; d < DPL; ++d) acc[g][d] *= corr;
    }
    const int n_here = min(32, end - base);
#pragma unroll 8
    for (int j = 0; j < n_here; ++j) {
      float vf[DPL];
      const half2* vh = reinterpret_cast<const half2*>(sV + j * RS + lane * DPL);
#pragma unroll
      for (int d = 0; d < DPL / 2; ++d) {
        const float2 f = __half22float2(vh[d]);
        vf[2 * d] = f.x;
        vf[2 * d + 1] = f.y;
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
#endif
  ATT_TP(3);
  __syncthreads();
  // merge the warps: four consecutive dims per thread (float4), the same
  // per-element summation order over warps as a scalar loop
#pragma unroll 1
  // (warps whose first tile lies past `end` hold no positions: skipped)
  const int w_act = min(W, (end - begin + PT - 1) / PT);
  for (int i = threadIdx.x; i < G * D / 4; i += blockDim.x) {
    const int g = i / (D / 4), d = (i % (D / 4)) * 4;
    float M = -INFINITY;
#pragma unroll 4
    for (int w = 0; w < w_act; ++w) M = fmaxf(M, wm[w][g]);
    float L = 0.0f;
    float4 A = make_float4(0.f, 0.f, 0.f, 0.f);
    if (M != -INFINITY) {
#pragma unroll 4
      for (int w = 0; w < w_act; ++w) {
        const float f = __expf(wm[w][g] - M);
        const float4 a = *reinterpret_cast<const float4*>(&wacc[w][g][d]);
        L += wl[w][g] * f;
        A.x += a.x * f;
        A.y += a.y * f;
        A.z += a.z * f;
        A.w += a.w * f;
      }
    }
    const int hq = hk * G + g;
    if (active == 1) {
      float4 r;
      r.x = L > 0.0f ? __fdividef(A.x, L) : 0.0f;
      r.y = L > 0.0f ? __fdividef(A.y, L) : 0.0f;
      r.z = L > 0.0f ? __fdividef(A.z, L) : 0.0f;
      r.w = L > 0.0f ? __fdividef(A.w, L) : 0.0f;
      *reinterpret_cast<float4*>(&o[(size_t(t) * Hq + hq) * D + d]) = r;
    } else {
      const size_t idx = (size_t(t) * Hq + hq) * nsplit + sp;
      *reinterpret_cast<float4*>(&part_o[idx * D + d]) = A;
      if (d == 0) {
        part_ml[idx * 2] = M;
        part_ml[idx * 2 + 1] = L;
      }
    }
  }
  ATT_TP(4);
  if (active == 1) return;
  // the last split to finish merges all partials of this (token, kv head)
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int done = atomicAdd(&counters[t * Hk + hk], 1);
    is_last = done == active - 1;
    if (is_last) counters[t * Hk + hk] = 0;  // self-reset for the next step
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
#pragma unroll 1
  for (int i = threadIdx.x; i < G * D; i += blockDim.x) {
    const int g = i / D, d = i % D;
    const size_t base = (size_t(t) * Hq + hk * G + g) * nsplit;
    float M = -INFINITY;
    for (int s2 = 0; s2 < active; ++s2) M = fmaxf(M, __ldcg(&part_ml[(base + s2) * 2]));
    float L = 0.0f, A = 0.0f;
    for (int s2 = 0; s2 < active; ++s2) {
      const float ms = __ldcg(&part_ml[(base + s2) * 2]);
      if (ms == -INFINITY) continue;
      const float f = __expf(ms - M);
      L += __ldcg(&part_ml[(base + s2) * 2 + 1]) * f;
      A += __ldcg(&part_o[(base + s2) * D + d]) * f;
    }
    o[(size_t(t) * Hq + hk * G + g) * D + d] = L > 0.0f ? __fdividef(A, L) : 0.0f;
  }
  ATT_TP(5);
}

__global__ void attn_combine_kernel(const float* __restrict__ part_o,
                                    const float* __restrict__ part_ml, const int* __restrict__ pos,
                                    int Hq, int D, int nsplit, float* __restrict__ o) {
  pdl_wait();
  pdl_trigger();
  const int t = blockIdx.x, hq = blockIdx.y;
  const int ctx = pos[t] + 1;
  const int chunk = split_chunk(ctx, nsplit);
  if (chunk >= ctx) return;  // single split wrote o directly
  const int active = (ctx + chunk - 1) / chunk;
  const size_t base = (size_t(t) * Hq + hq) * nsplit;
  float M = -INFINITY;
  for (int s = 0; s < active; ++s) M = fmaxf(M, part_ml[(base + s) * 2]);
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    float L = 0.0f, A = 0.0f;
    for (int s = 0; s < active; ++s) {
      const float ms = part_ml[(base + s) * 2];
      if (ms == -INFINITY) continue;
      const float f = expf(ms - M);
      L += part_ml[(base + s) * 2 + 1] * f;
      A += part_o[(base + s) * D + d] * f;
    }
    o[(size_t(t) * Hq + hq) * D + d] = L > 0.0f ? A / L : 0.0f;
  }
}

template <int D, bool FUSED>
void attn_d(int G, dim3 grid, const half* q, const float* qkv, const float* inv_freq,
            const int* pos, const int* slot, const int* seq_of, const int* bt, int maxb, half* kc,
            half* vc, int Hq, int Hk, int nsplit, float* po, float* pml, float* o,
            cudaStream_t st) {
  const dim3 thr(kAttnWarps * 32);
  const size_t smem = size_t(kAttnWarps) * 32 * (D + kKvPad) * sizeof(half);
#define MSW_ATT(GG)                                                                              \
  case GG: {                                                                                     \
    static bool attr = false;                                                                    \
    if (!attr) {                                                                                 \
      MSW_CUDA(cudaFuncSetAttribute(attention_kernel<D, GG, FUSED>,                              \
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));    \
      attr = true;                                                                               \
    }                                                                                            \
    launch_pdl(attention_kernel<D, GG, FUSED>, grid, thr, smem, st, q, qkv, inv_freq, pos, slot, \
               seq_of, bt, maxb, kc, vc, Hq, Hk, nsplit, po, pml, o);                            \
    break;                                                                                       \
  }
  switch (G) {
    MSW_ATT(1)
    MSW_ATT(2)
    MSW_ATT(4)
    MSW_ATT(8)
    default: throw ConfigErr("attention: GQA group must be 1, 2, 4 or 8");
  }
#undef MSW_ATT
}

template <bool FUSED>
void attention_any(const half* q, const float* qkv, const float* inv_freq, int T, const int* pos,
                   const int* slot, const int* seq_of, const int* block_table, half* kc, half* vc,
                   const AttnShape& a, int nsplit, float* part_o, float* part_ml, float* o,
                   cudaStream_t st) {
  const int G = a.n_heads / a.n_kv_heads;
  const dim3 grid(T, a.n_kv_heads, nsplit);
  if (a.head_dim == 128)
    attn_d<128, FUSED>(G, grid, q, qkv, inv_freq, pos, slot, seq_of, block_table,
                       a.max_blocks_per_seq, kc, vc, a.n_heads, a.n_kv_heads, nsplit, part_o,
                       part_ml, o, st);
  else if (a.head_dim == 64)
    attn_d<64, FUSED>(G, grid, q, qkv, inv_freq, pos, slot, seq_of, block_table,
                      a.max_blocks_per_seq, kc, vc, a.n_heads, a.n_kv_heads, nsplit, part_o,
                      part_ml, o, st);
  else
    throw ConfigErr("attention: head_dim must be 64 or 128");
  if (nsplit > 1)
    launch_pdl(attn_combine_kernel, dim3(T, a.n_heads), dim3(128), 0, st, part_o, part_ml, pos,
               a.n_heads, a.head_dim, nsplit, o);
}

}  // namespace

void launch_rope_table(const float* inv_freq, int head_dim, int max_pos, float2* table,
                       cudaStream_t st) {
  rope_table_kernel<<<kNumSMs * 4, 256, 0, st>>>(inv_freq, head_dim / 2, max_pos, table);
  MSW_LAUNCH_CHECK();
}

void launch_rope_append(const float* qkv, int T, const int* pos, const int* slot,
                        const float2* rope, const AttnShape& a, half* q_out, half* kc, half* vc,
                        cudaStream_t st) {
  launch_pdl(rope_append_kernel, dim3(T), dim3(256), 0, st, qkv, pos, slot, rope, a.n_heads,
             a.n_kv_heads, a.head_dim, q_out, kc, vc);
}

void launch_attention(const half* q, int T, const int* pos, const int* seq_of,
                      const int* block_table, const half* kc, const half* vc, const AttnShape& a,
                      int nsplit, float* part_o, float* part_ml, float* o, cudaStream_t st) {
  attention_any<false>(q, nullptr, nullptr, T, pos, nullptr, seq_of, block_table,
                       const_cast<half*>(kc), const_cast<half*>(vc), a, nsplit, part_o, part_ml, o,
                       st);
}

template <bool KV8>
void launch_attention_decode_t(const float* qkv, const float2* rope, int T, const int* pos,
                               const int* slot, const int* seq_of, const int* block_table,
                               typename std::conditional<KV8, uint8_t, half>::type* kc,
                               typename std::conditional<KV8, uint8_t, half>::type* vc,
                               const AttnShape& a, int nsplit, float* part_o, float* part_ml,
                               int* counters, float* o, cudaStream_t st, bool run) {
  const int G = a.n_heads / a.n_kv_heads;
  if (run && T > kRunMax) throw ConfigErr("attention: a one-sequence run is at most 6 tokens");
  const dim3 grid(T, a.n_kv_heads, nsplit);
  // many (token, kv head, split) CTAs (continuous batching): 4-warp CTAs use
  // 70 KB of staging instead of 139 KB, so three are resident per SM and more
  // KV is in flight; a few CTAs (batch-1 decode): 8 warps for latency
  const bool wide = size_t(T) * a.n_kv_heads * nsplit >= size_t(2) * kNumSMs;
  // (16 warps x 16-position tiles for batch-1 decode measured 1% slower per
  // token than 8 warps x 32 positions: 1.464-1.477 vs 1.442-1.456 ms, 8B W4)
#define MSW_DEC_W(DD, GG, WW, PP)                                                                 \
  {                                                                                               \
    const size_t smem = size_t(WW) * 2 * PP * (DD + kKvPad) * sizeof(half);                      \
    static bool attr = false;                                                                     \
    if (!attr) {                                                                                  \
      MSW_CUDA(cudaFuncSetAttribute(attn_decode_kernel<DD, GG, WW, KV8, PP>,                      \
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));     \
      attr = true;                                                                                \
    }                                                                                             \
    return launch_pdl(attn_decode_kernel<DD, GG, WW, KV8, PP>, grid, dim3(WW * 32), smem, st, qkv, \
                      rope, pos, slot, seq_of, block_table, a.max_blocks_per_seq, kc, vc,         \
                      a.n_heads, a.n_kv_heads, nsplit, part_o, part_ml, counters, o,              \
                      run ? 1 : 0);                                                               \
  }
#define MSW_DEC(DD, GG)                                                  \
  if (a.head_dim == DD && G == GG) {                                     \
    if (wide) MSW_DEC_W(DD, GG, 4, 32)                                   \
    MSW_DEC_W(DD, GG, 8, 32)                                             \
  }
  MSW_DEC(128, 1)
  MSW_DEC(128, 2)
  MSW_DEC(128, 4)
  MSW_DEC(128, 8)
  MSW_DEC(64, 1)
  MSW_DEC(64, 2)
  MSW_DEC(64, 4)
  MSW_DEC(64, 8)
#undef MSW_DEC
#undef MSW_DEC_W
  throw ConfigErr("attention: unsupported head_dim / GQA group");
}

__global__ void kv_compress_kernel(const half* __restrict__ kc, const half* __restrict__ vc,
                                   uint8_t* __restrict__ kc8, uint8_t* __restrict__ vc8,
                                   size_t layer_elems, const int* __restrict__ b16,
                                   const int* __restrict__ b8, int Hk, int D) {
  const int p = blockIdx.x, l = blockIdx.y;
  const int s16 = b16[p >> 4] * kKvBlock + (p & 15), s8 = b8[p >> 4] * kKvBlock + (p & 15);
  const size_t lo = size_t(l) * layer_elems;
  for (int i = threadIdx.x; i < Hk * D / 2; i += blockDim.x) {
    const int hk = (2 * i) / D, d = (2 * i) % D;
    const size_t a = lo + kv_off(s16, hk, Hk, D) + d, b = lo + kv_off(s8, hk, Hk, D) + d;
    *reinterpret_cast<uint16_t*>(kc8 + b) = h2_to_e4m3x2(kc[a], kc[a + 1]);
    *reinterpret_cast<uint16_t*>(vc8 + b) = h2_to_e4m3x2(vc[a], vc[a + 1]);
  }
}

__global__ void fp8_roundtrip_kernel(const half* __restrict__ x, int64_t n, uint8_t* __restrict__ q,
                                     half* __restrict__ y) {
  for (int64_t i = 2 * (blockIdx.x * int64_t(blockDim.x) + threadIdx.x); i + 1 < n;
       i += 2 * int64_t(gridDim.x) * blockDim.x) {
    const uint16_t v = h2_to_e4m3x2(x[i], x[i + 1]);
    *reinterpret_cast<uint16_t*>(q + i) = v;
    *reinterpret_cast<uint32_t*>(y + i) = e4m3x2_to_h2(v);
  }
}

void launch_attention_decode(const float* qkv, const float2* rope, int T, const int* pos,
                             const int* slot, const int* seq_of, const int* block_table, half* kc,
                             half* vc, const AttnShape& a, int nsplit, float* part_o,
                             float* part_ml, int* counters, float* o, cudaStream_t st, bool run) {
  launch_attention_decode_t<false>(qkv, rope, T, pos, slot, seq_of, block_table, kc, vc, a, nsplit,
                                   part_o, part_ml, counters, o, st, run);
}

void launch_attention_decode_kv8(const float* qkv, const float2* rope, int T, const int* pos,
                                 const int* slot, const int* seq_of, const int* block_table,
                                 uint8_t* kc, uint8_t* vc, const AttnShape& a, int nsplit,
                                 float* part_o, float* part_ml, int* counters, float* o,
                                 cudaStream_t st, bool run) {
  launch_attention_decode_t<true>(qkv, rope, T, pos, slot, seq_of, block_table, kc, vc, a, nsplit,
                                  part_o, part_ml, counters, o, st, run);
}

void launch_kv_compress(const half* kc, const half* vc, uint8_t* kc8, uint8_t* vc8,
                        size_t layer_elems, int layers, const int* b16, const int* b8, int npos,
                        int Hk, int D, cudaStream_t st) {
  if (npos <= 0) return;
  kv_compress_kernel<<<dim3(npos, layers), 256, 0, st>>>(kc, vc, kc8, vc8, layer_elems, b16, b8, Hk, D);
  MSW_CUDA(cudaGetLastError());
}

void launch_fp8_roundtrip(const half* x, int64_t n, uint8_t* q, half* y, cudaStream_t st) {
  if (n <= 0) return;
  const int grid = int(std::min<int64_t>((n / 2 + 255) / 256, 4 * kNumSMs));
  fp8_roundtrip_kernel<<<std::max(grid, 1), 256, 0, st>>>(x, n, q, y);
  MSW_CUDA(cudaGetLastError());
}

}  // namespace msw
