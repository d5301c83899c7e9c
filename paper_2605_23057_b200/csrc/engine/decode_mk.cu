// Persistent batch-1 decode step: the whole token (embedding, every layer's
// RMSNorm + QKV / RoPE + KV append + attention / O + residual / RMSNorm +
// gate_up + SwiGLU / down + residual, final norm + lm_head, greedy argmax and
// the position advance) in ONE launch of one CTA per SM.
//
// Why: as separate kernels, every GEMV CTA owns its SM (190 KB smem, 576
// threads), so the next kernel's CTAs cannot become resident until the
// current one exits and the weight stream stalls at each of the ~164 kernel
// boundaries per token (activation prologue + ring refill + tail, 2-4 us each;
// measured with scripts/gemv_timeline.py). Here the producer warp of every SM
// streams its share of ALL weight matrices of the step back to back through
// one cp.async.bulk ring, never waiting on activations; only the consumers
// wait, on grid-wide phase barriers, so barrier and attention latency hide
// behind the ring (5 x 32 KB per SM = 24 MB in flight chip-wide).
//
// Roles per CTA (576 threads, 1 CTA per SM, grid = 148):
//   warps 0..15  consumers: per GEMV phase, wait for the input barrier, stage
//                the activation (RMSNorm, fp16 / int8 / fp16 + W4 group
//                offsets), then run mma.sync over the ring; attention phases
//                and the embedding run on these warps too;
//   warp 16      producer: scales + weight stages of every GEMV phase, in order;
//   warp 17      epilogue: per 16-row tile, sums the 16 warps' partials, applies
//                INT8 scales / SwiGLU / residual / logits + argmax, stores,
//                and arrives on the phase barrier.
// Weight formats and numerics are those of the per-kernel decode path
// (gemv.cu, attention.cu, misc.cu), except the W4 nibble extraction: all four
// k16 steps use (1024 + q) against x (shifts on the FMA pipe via mul.hi), and
// the per-group offset is 1032 * sum(x_group).
#include <algorithm>
#include <type_traits>

#include "kernels.cuh"
#include "mma_frag.cuh"

namespace msw {
namespace {

constexpr int kMkCons = 16;
constexpr int kMkThreads = (kMkCons + 2) * 32;
constexpr int kMkConsThreads = kMkCons * 32;
constexpr int kMkCPW = 4;                       // chunks per warp per stage
constexpr int kMkMaxS = kMkCons * kMkCPW;       // 64 chunks of 512 B
constexpr int kMkSlotBytes = kMkMaxS * 512;     // 32 KB ring slot
constexpr int kMkMaxSlots = 8;
constexpr int kMkXRegs = 8;                     // float4 of x per thread (k <= 16384)
constexpr int kMkAttnMinChunk = 64;             // positions per attention split, at least
constexpr int kBarNamedCons = 1;                // named barrier: consumers
constexpr int kBarNamedHand = 3;                // named barrier: consumers + epilogue

enum MkEpi { kMkStore = 0, kMkResid = 1, kMkSwiglu = 2, kMkHead = 3 };

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned long long mk_amax_key(float v, int i) {
  const uint32_t u = __float_as_uint(v);
  const uint32_t o = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return (static_cast<unsigned long long>(o) << 32) | (0xFFFFFFFFu - uint32_t(i));
}

struct MkShared {
  uint64_t full[kMkMaxSlots], empty[kMkMaxSlots];
  uint64_t sc_full[2], sc_empty[2];
  uint64_t tile_full[2], tile_free[2];
  float part[2][kMkCons][16];
  float red[32];
  float xscale;
  int attn_last;
  unsigned target_base;
  int tok, pos, slot, step;
};

// Per-CTA slice of one linear for this step.
struct Slice {
  int ct;       // chunks per 16-row tile
  int S;        // chunks per stage (min(64, ct))
  int tb, nt;   // first tile, tile count
  int total;    // chunks in this CTA's stream
  int stages;
};

__device__ __forceinline__ int chunk_k(int fmt) { return fmt == kFP16 ? 16 : (fmt == kINT8 ? 32 : 64); }

__device__ __forceinline__ Slice make_slice(const MkLinear& L, int fmt) {
  Slice s;
  s.ct = L.k / chunk_k(fmt);
  s.S = min(kMkMaxS, s.ct);
  const int ntiles = L.n / 16;
  const int per = (ntiles + gridDim.x - 1) / gridDim.x;
  s.tb = min(ntiles, int(blockIdx.x) * per);
  s.nt = max(0, min(ntiles, s.tb + per) - s.tb);
  s.total = s.nt * s.ct;
  s.stages = (s.total + s.S - 1) / s.S;
  return s;
}
__device__ __forceinline__ int scale_bytes(const MkLinear& L, int fmt, const Slice& s) {
  return fmt == kW4 ? s.nt * 16 * (L.k / kW4Group) * 2 : (fmt == kINT8 ? s.nt * 16 * 4 : 0);
}

// ------------------------------------------------------------------ barrier
// Monotonic arrival counter; barrier j of launch e completes at
// (e * n_bar + j + 1) * gridDim.x arrivals (u32, wrap-safe compare). The
// launch counter `epoch` is read by every CTA at start and bumped by CTA 0
// after the last barrier, so no reset races exist.
__device__ __forceinline__ void grid_arrive(const MkParams& P) {
  __threadfence();
  red_release_add(P.bar, 1u);
}
__device__ __forceinline__ void grid_wait(const MkParams& P, const MkShared& sh, int j) {
  const unsigned target = sh.target_base + unsigned(j + 1) * gridDim.x;
  while (int(ld_acquire_u32(P.bar) - target) < 0) {
  }
}

// --------------------------------------------------------------- prologue
// x fp32 [k] (global, written by earlier phases) -> xs (smem):
//   FP16: fp16 [k] permuted (perm_f16); INT8: int8 [k] permuted (perm_i8) +
//   sh.xscale; W4: fp16 [k] permuted + float corr[k/128] = 1032 * sum(x_group).
// Thread t handles float4 i = t + 512 j (registers between the passes); warp w
// covers k in [128 (w + 16 j), +128) = one W4 scale group per j.
template <int FMT, bool NORM>
__device__ __noinline__ void mk_prologue(const float* __restrict__ x,
                                            const half* __restrict__ gamma, float eps, int k,
                                            uint8_t* xs, MkShared& sh) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k4 = k >> 2;
  const float4* xt = reinterpret_cast<const float4*>(x);
  float4 v[kMkXRegs];
#pragma unroll
  for (int j = 0; j < kMkXRegs; ++j)
    if (tid + j * kMkConsThreads < k4) v[j] = __ldcg(xt + tid + j * kMkConsThreads);
  auto sync_red = [&](float val, bool is_max) -> float {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float t = __shfl_xor_sync(0xffffffffu, val, o);
      val = is_max ? fmaxf(val, t) : val + t;
    }
    named_sync(kBarNamedCons, kMkConsThreads);
    if (lane == 0) sh.red[warp] = val;
    named_sync(kBarNamedCons, kMkConsThreads);
    float t = lane < kMkCons ? sh.red[lane] : (is_max ? -3.402823466e38f : 0.0f);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float u = __shfl_xor_sync(0xffffffffu, t, o);
      t = is_max ? fmaxf(t, u) : t + u;
    }
    return t;
  };
  if (NORM) {
    float ss = 0.0f;
#pragma unroll
    for (int j = 0; j < kMkXRegs; ++j)
      if (tid + j * kMkConsThreads < k4)
        ss = fmaf(v[j].x, v[j].x, fmaf(v[j].y, v[j].y, fmaf(v[j].z, v[j].z, fmaf(v[j].w, v[j].w, ss))));
    ss = sync_red(ss, false);
    const float r = 1.0f / sqrtf(ss / float(k) + eps);
#pragma unroll
    for (int j = 0; j < kMkXRegs; ++j) {
      const int i = tid + j * kMkConsThreads;
      if (i < k4) {
        const half2* gm = reinterpret_cast<const half2*>(gamma) + 2 * i;
        const float2 g0 = __half22float2(gm[0]), g1 = __half22float2(gm[1]);
        v[j].x = (v[j].x * r) * g0.x;
        v[j].y = (v[j].y * r) * g0.y;
        v[j].z = (v[j].z * r) * g1.x;
        v[j].w = (v[j].w * r) * g1.y;
      }
    }
  }
  if (FMT == kINT8) {
    float amax = 0.0f;
#pragma unroll
    for (int j = 0; j < kMkXRegs; ++j)
      if (tid + j * kMkConsThreads < k4)
        amax = fmaxf(amax, fmaxf(fmaxf(fabsf(v[j].x), fabsf(v[j].y)), fmaxf(fabsf(v[j].z), fabsf(v[j].w))));
    amax = sync_red(amax, true);
    const float s = amax / 127.0f;
    auto q = [&](float val) -> int8_t {
      const float u = amax > 0.0f ? rintf(val / s) : 0.0f;
      return static_cast<int8_t>(fminf(fmaxf(u, -127.0f), 127.0f));
    };
    int8_t* xq = reinterpret_cast<int8_t*>(xs);
#pragma unroll
    for (int j = 0; j < kMkXRegs; ++j) {
      const int i = tid + j * kMkConsThreads;
      if (i < k4)
        *reinterpret_cast<char4*>(xq + perm_i8(4 * i)) = make_char4(q(v[j].x), q(v[j].y), q(v[j].z), q(v[j].w));
    }
    if (tid == 0) sh.xscale = s;
  } else {
    half* xh = reinterpret_cast<half*>(xs);
    float* corr = reinterpret_cast<float*>(xs + size_t(2) * k);
#pragma unroll
    for (int j = 0; j < kMkXRegs; ++j) {
      const int i = tid + j * kMkConsThreads;
      if (warp * 32 + j * kMkConsThreads >= k4) continue;  // warp-uniform (k4 % 32 == 0)
      const half2 lo = __floats2half2_rn(v[j].x, v[j].y), hi = __floats2half2_rn(v[j].z, v[j].w);
      *reinterpret_cast<half2*>(xh + perm_f16(4 * i)) = lo;
      *reinterpret_cast<half2*>(xh + perm_f16(4 * i + 2)) = hi;
      if (FMT == kW4) {
        const float2 lf = __half22float2(lo), hf = __half22float2(hi);
        float gs = (lf.x + lf.y) + (hf.x + hf.y);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) gs += __shfl_xor_sync(0xffffffffu, gs, o);
        if (lane == 0) corr[warp + j * kMkCons] = 1032.0f * gs;
      }
    }
  }
  named_sync(kBarNamedCons, kMkConsThreads);
}

// ------------------------------------------------------------ GEMV consumer
// One linear's share of this CTA: stages of S chunks from the ring; warp w
// takes chunks [4w, 4w + 4) of each stage. Every consumer warp flushes every
// tile exactly once, in order (zero partial if it never touched it).
template <int FMT, bool XREG>
__device__ __noinline__ void mk_consume(const Slice& sl, int groups_k, const uint8_t* xs,
                                           const uint8_t* ring, const half* sc_h, int n_slots,
                                           int& slot, uint32_t& phase, int& tile_ctr,
                                           MkShared& sh, uint32_t one) {
  using Acc = typename std::conditional<FMT == kINT8, int, float>::type;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  const uint8_t* xrow = xs + tq * 8;  // batch-1: every MMA column reads token 0
  const float* corr = reinterpret_cast<const float*>(xs + size_t(sl.ct) * 64 * 2);
  const int w0c = warp * kMkCPW;      // this warp's chunk offset inside a stage
  uint2 bx[XREG ? kMkCPW : 1][2][2];
  float cx[XREG ? 2 : 1];
  if (XREG) {  // W4, one tile per stage: the k-slice never moves
#pragma unroll
    for (int j = 0; j < kMkCPW; ++j)
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const int kb = ((w0c + j) * 64 + p * 32) * 2;
        bx[XREG ? j : 0][p][0] = *reinterpret_cast<const uint2*>(xrow + kb);
        bx[XREG ? j : 0][p][1] = *reinterpret_cast<const uint2*>(xrow + kb + 32);
      }
    cx[0] = corr[w0c / 2];
    cx[XREG ? 1 : 0] = corr[w0c / 2 + 1];
  }
  const uint32_t shr4 = one << 28, shr8 = one << 24, shr12 = one << 20;
  Acc acc[4] = {0, 0, 0, 0};
  int ti = 0;                    // next tile to flush (CTA-local)
  int ts = w0c / sl.ct;          // tile of this warp's slice in the current stage
  int cs = w0c - ts * sl.ct;     // chunk offset of the slice inside that tile
  auto flush = [&]() {
    const int b = tile_ctr & 1;
    if (tile_ctr >= 2) mbar_wait(&sh.tile_free[b], ((tile_ctr >> 1) - 1) & 1);
    if (tq == 0) {
      float* pw = &sh.part[b][warp][0];
      pw[g] = FMT == kINT8 ? __int_as_float(int(acc[0])) : float(acc[0]);
      pw[g + 8] = FMT == kINT8 ? __int_as_float(int(acc[2])) : float(acc[2]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sh.tile_full[b]);
    acc[0] = acc[1] = acc[2] = acc[3] = 0;
    ++tile_ctr;
    ++ti;
  };
#pragma unroll 1
  for (int st = 0; st < sl.stages; ++st) {
    const int stage_chunks = min(sl.S, sl.total - st * sl.S);
    const bool active = w0c < stage_chunks;
    if (active) {
      while (ti < ts) flush();
    }
    mbar_wait(&sh.full[slot], phase);
    uint4 a4[kMkCPW];
    if (active) {
      const uint4* stg = reinterpret_cast<const uint4*>(ring + size_t(slot) * kMkSlotBytes) + w0c * 32 + lane;
#pragma unroll
      for (int j = 0; j < kMkCPW; ++j) a4[j] = stg[j * 32];
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sh.empty[slot]);
    if (++slot == n_slots) {
      slot = 0;
      phase ^= 1;
    }
    if (active) {
      if constexpr (FMT == kFP16) {
        float acc2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int j = 0; j < kMkCPW; ++j) {
          const uint2 b = *reinterpret_cast<const uint2*>(xrow + (cs + j) * 32);
          const uint32_t a[4] = {a4[j].x, a4[j].y, a4[j].z, a4[j].w};
          mma_f16((j & 1) ? acc2 : reinterpret_cast<float(&)[4]>(acc), a, b.x, b.y);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i] += acc2[i];
      } else if constexpr (FMT == kINT8) {
        int acc2[4] = {0, 0, 0, 0};
#pragma unroll
        for (int j = 0; j < kMkCPW; ++j) {
          const uint2 b = *reinterpret_cast<const uint2*>(xrow + (cs + j) * 32);
          const uint32_t a[4] = {a4[j].x, a4[j].y, a4[j].z, a4[j].w};
          mma_s8((j & 1) ? acc2 : reinterpret_cast<int(&)[4]>(acc), a, b.x, b.y);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i] += acc2[i];
      } else {
        const int lr = (ts - 0) * 16 + g;  // local row (tile-local index ts)
#pragma unroll
        for (int jj = 0; jj < kMkCPW / 2; ++jj) {
          float cg[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int j = 2 * jj; j < 2 * jj + 2; ++j) {
            const uint32_t wv[4] = {a4[j].x, a4[j].y, a4[j].z, a4[j].w};
#pragma unroll
            for (int p = 0; p < 2; ++p) {
              const uint32_t w0 = wv[2 * p], w1 = wv[2 * p + 1];
              // nibble positions 0/4 (step 2p, row g), 2/6 (step 2p, row g+8),
              // 1/5 (step 2p+1, row g), 3/7 (step 2p+1, row g+8): shifts on the FMA pipe
              const uint32_t a_lo[4] = {lop3_and_or(w0, 0x000F000Fu, 0x64006400u),
                                        lop3_and_or(__umulhi(w0, shr8), 0x000F000Fu, 0x64006400u),
                                        lop3_and_or(w1, 0x000F000Fu, 0x64006400u),
                                        lop3_and_or(__umulhi(w1, shr8), 0x000F000Fu, 0x64006400u)};
              const uint32_t a_hi[4] = {lop3_and_or(__umulhi(w0, shr4), 0x000F000Fu, 0x64006400u),
                                        lop3_and_or(__umulhi(w0, shr12), 0x000F000Fu, 0x64006400u),
                                        lop3_and_or(__umulhi(w1, shr4), 0x000F000Fu, 0x64006400u),
                                        lop3_and_or(__umulhi(w1, shr12), 0x000F000Fu, 0x64006400u)};
              uint2 be, bo;
              if (XREG) {
                be = bx[XREG ? j : 0][p][0];
                bo = bx[XREG ? j : 0][p][1];
              } else {
                const int kb = ((cs + j) * 64 + p * 32) * 2;
                be = *reinterpret_cast<const uint2*>(xrow + kb);
                bo = *reinterpret_cast<const uint2*>(xrow + kb + 32);
              }
              mma_f16(cg, a_lo, be.x, be.y);
              mma_f16(cg, a_hi, bo.x, bo.y);
            }
          }
          const int grp = (cs >> 1) + jj;
          const float slo = __half2float(sc_h[lr * groups_k + grp]);
          const float shi = __half2float(sc_h[(lr + 8) * groups_k + grp]);
          const float c = XREG ? cx[XREG ? jj : 0] : corr[grp];
          acc[0] = fmaf(slo, cg[0] - c, acc[0]);
          acc[2] = fmaf(shi, cg[2] - c, acc[2]);
        }
      }
    }
    // advance the slice by one stage; tiles that ended inside this stage are done
    cs += sl.S;
    if (cs >= sl.ct) {
      cs -= sl.ct;
      ++ts;
    }
    const int stage_end = (st + 1) * sl.S;
    if (!active || ts > ti) {
      while (ti < sl.nt && (ti + 1) * sl.ct <= stage_end && ti < ts) flush();
    }
    if (!active) {
      while (ti < sl.nt && (ti + 1) * sl.ct <= stage_end) flush();
    }
  }
  while (ti < sl.nt) flush();
}

// ---------------------------------------------------------- GEMV epilogue
template <int FMT, int EPI>
__device__ __noinline__ void mk_epilogue(const Slice& sl, const MkLinear& L, const uint8_t* sc,
                                            float* y, int& tile_ctr, MkShared& sh,
                                            unsigned long long& best) {
  const int lane = threadIdx.x & 31;
  for (int i = 0; i < sl.nt; ++i) {
    const int b = tile_ctr & 1;
    mbar_wait(&sh.tile_full[b], (tile_ctr >> 1) & 1);
    const int row = (sl.tb + i) * 16 + (lane & 15);
    float v = 0.0f;
    if (FMT == kINT8) {
      int iv = 0;
#pragma unroll
      for (int w = 0; w < kMkCons; ++w) iv += __float_as_int(sh.part[b][w][lane & 15]);
      v = (float(iv) * sh.xscale) * reinterpret_cast<const float*>(sc)[i * 16 + (lane & 15)];
    } else {
#pragma unroll
      for (int w = 0; w < kMkCons; ++w) v += sh.part[b][w][lane & 15];
    }
    if (EPI == kMkSwiglu) {
      const float u = __shfl_down_sync(0xffffffffu, v, 1);  // rows (2i, 2i+1) = (gate_i, up_i)
      if (lane < 16 && (lane & 1) == 0) y[row / 2] = silu(v) * u;
    } else if (lane < 16) {
      if (EPI == kMkStore) y[row] = v;
      if (EPI == kMkResid) y[row] = __ldcg(y + row) + v;
      if (EPI == kMkHead) {
        y[row] = v;
        const unsigned long long kk = mk_amax_key(v, row);
        best = kk > best ? kk : best;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sh.tile_free[b]);
    ++tile_ctr;
  }
}

// -------------------------------------------------------------- attention
// Decode attention of one layer for the (single) new token at position p.
// Work items (kv head hk, split sp) map to CTAs; each CTA: RoPE of its G query
// heads and the new key (table lookup, as attention.cu), split 0 appends k/v
// to the paged cache, 16 warps x 32 positions per pass (lane = position, K/V
// rows read straight from the cache), in-CTA merge through shared memory, and
// across splits the last CTA of a head (counter) merges the partials.
template <int D, int G>
__device__ __noinline__ void mk_attention(const MkParams& P, const MkLayer& Ly, uint8_t* xs, MkShared& sh) {
  constexpr int DPL = D / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int Hq = P.Hq, Hk = P.Hk;
  const int p_self = sh.pos, ctx = p_self + 1;
  int nsplit = min(P.nsplit_max, max(1, int(gridDim.x) / Hk));
  nsplit = min(nsplit, max(1, (ctx + kMkAttnMinChunk - 1) / kMkAttnMinChunk));
  int chunk = (ctx + nsplit - 1) / nsplit;
  chunk = ((chunk + 31) / 32) * 32;
  const int active = (ctx + chunk - 1) / chunk;
  const int item = blockIdx.x;
  if (item >= Hk * active) return;
  const int hk = item % Hk, sp = item / Hk;
  const int begin = sp * chunk, end = min(ctx, begin + chunk);
  // smem carve-up (xs region): qs[G][D] f32 | knew[D], vnew[D] f16 | wm, wl [16][G] | wacc [16][G][D]
  float* qs = reinterpret_cast<float*>(xs);
  half* knew = reinterpret_cast<half*>(qs + G * D);
  half* vnew = knew + D;
  float* wm = reinterpret_cast<float*>(vnew + D);
  float* wl = wm + kMkCons * G;
  float* wacc = wl + kMkCons * G;
  const float* row = P.qkv;
  const float2* rp = P.rope + size_t(p_self) * (D / 2);
  for (int i = tid; i < (G + 1) * (D / 2); i += kMkConsThreads) {
    const int h = i / (D / 2), j = i % (D / 2);
    const float* src = h < G ? row + size_t(hk * G + h) * D : row + size_t(Hq + hk) * D;
    const float2 r = rp[j];
    const float x0 = __ldcg(src + j), x1 = __ldcg(src + j + D / 2);
    const half y0 = __float2half_rn(__fsub_rn(__fmul_rn(x0, r.x), __fmul_rn(x1, r.y)));
    const half y1 = __float2half_rn(__fadd_rn(__fmul_rn(x1, r.x), __fmul_rn(x0, r.y)));
    if (h < G) {
      qs[h * D + j] = __half2float(y0);
      qs[h * D + j + D / 2] = __half2float(y1);
    } else {
      knew[j] = y0;
      knew[j + D / 2] = y1;
    }
  }
  for (int d = tid; d < D; d += kMkConsThreads)
    vnew[d] = __float2half_rn(__ldcg(row + size_t(Hq + Hk + hk) * D + d));
  named_sync(kBarNamedCons, kMkConsThreads);
  half* kc = Ly.kc;
  half* vc = Ly.vc;
  auto kv_off = [&](int s) { return ((size_t(s >> 4) * Hk + hk) * 16 + (s & 15)) * size_t(D); };
  if (sp == 0)
    for (int d = tid; d < D; d += kMkConsThreads) {
      kc[kv_off(sh.slot) + d] = knew[d];
      vc[kv_off(sh.slot) + d] = vnew[d];
    }
  const float scale = rsqrtf(float(D));
  float m[G], l[G], acc[G][DPL];
#pragma unroll
  for (int gg = 0; gg < G; ++gg) {
    m[gg] = -INFINITY;
    l[gg] = 0.0f;
#pragma unroll
    for (int d = 0; d < DPL; ++d) acc[gg][d] = 0.0f;
  }
  const int* bt = P.block_table;  // batch-1 decode: row 0
#pragma unroll 1
  for (int base = begin + warp * 32; base < end; base += kMkCons * 32) {
    const int p = base + lane;
    const bool valid = p < end;
    int sl_p = 0;
    if (valid && p != p_self) sl_p = bt[p >> 4] * 16 + (p & 15);
    float s[G];
#pragma unroll
    for (int gg = 0; gg < G; ++gg) s[gg] = 0.0f;
    if (valid) {
      const uint4* kr = p == p_self ? reinterpret_cast<const uint4*>(knew)
                                    : reinterpret_cast<const uint4*>(kc + kv_off(sl_p));
#pragma unroll
      for (int c0 = 0; c0 < D / 8; c0 += 8) {
        uint4 kv[8];
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (c0 + c < D / 8) kv[c] = p == p_self ? kr[c0 + c] : __ldcg(kr + c0 + c);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          if (c0 + c >= D / 8) break;
          const half2* kh = reinterpret_cast<const half2*>(&kv[c]);
          const float2 k0 = __half22float2(kh[0]), k1 = __half22float2(kh[1]);
          const float2 k2 = __half22float2(kh[2]), k3 = __half22float2(kh[3]);
#pragma unroll
          for (int gg = 0; gg < G; ++gg) {
            const float4 q0 = *reinterpret_cast<const float4*>(&qs[gg * D + (c0 + c) * 8]);
            const float4 q1 = *reinterpret_cast<const float4*>(&qs[gg * D + (c0 + c) * 8 + 4]);
            s[gg] = fmaf(q0.x, k0.x, fmaf(q0.y, k0.y, fmaf(q0.z, k1.x, fmaf(q0.w, k1.y, s[gg]))));
            s[gg] = fmaf(q1.x, k2.x, fmaf(q1.y, k2.y, fmaf(q1.z, k3.x, fmaf(q1.w, k3.y, s[gg]))));
          }
        }
      }
    }
    float e[G];
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
      const float sv = valid ? s[gg] * scale : -INFINITY;
      const float mn = fmaxf(m[gg], warp_max(sv));
      const float corr = __expf(m[gg] - mn);
      e[gg] = valid ? __expf(sv - mn) : 0.0f;
      l[gg] = l[gg] * corr + warp_sum(e[gg]);
      m[gg] = mn;
#pragma unroll
      for (int d = 0; d < DPL; ++d) acc[gg][d] *= corr;
    }
    const int n_here = min(32, end - base);
#pragma unroll 4
    for (int j = 0; j < n_here; ++j) {
      const int pj = base + j;
      const half* vrow;
      if (pj == p_self) {
        vrow = vnew;
      } else {
        const int sj = __shfl_sync(0xffffffffu, sl_p, j);
        vrow = vc + kv_off(sj);
      }
      float vf[DPL];
      if (DPL == 4) {
        const uint2 u = pj == p_self ? *reinterpret_cast<const uint2*>(vrow + lane * 4)
                                     : __ldcg(reinterpret_cast<const uint2*>(vrow + lane * 4));
        const float2 f0 = __half22float2(*reinterpret_cast<const half2*>(&u.x));
        const float2 f1 = __half22float2(*reinterpret_cast<const half2*>(&u.y));
        vf[0] = f0.x;
        vf[1] = f0.y;
        vf[DPL > 2 ? 2 : 0] = f1.x;
        vf[DPL > 3 ? 3 : 0] = f1.y;
      } else {
        const unsigned u = pj == p_self ? *reinterpret_cast<const unsigned*>(vrow + lane * 2)
                                        : __ldcg(reinterpret_cast<const unsigned*>(vrow + lane * 2));
        const float2 f0 = __half22float2(*reinterpret_cast<const half2*>(&u));
        vf[0] = f0.x;
        vf[DPL > 1 ? 1 : 0] = f0.y;
      }
#pragma unroll
      for (int gg = 0; gg < G; ++gg) {
        const float w = __shfl_sync(0xffffffffu, e[gg], j);
#pragma unroll
        for (int d = 0; d < DPL; ++d) acc[gg][d] = fmaf(w, vf[d], acc[gg][d]);
      }
    }
  }
  // merge the 16 warps
#pragma unroll
  for (int gg = 0; gg < G; ++gg) {
    if (lane == 0) {
      wm[warp * G + gg] = m[gg];
      wl[warp * G + gg] = l[gg];
    }
#pragma unroll
    for (int d = 0; d < DPL; ++d) wacc[(warp * G + gg) * D + lane * DPL + d] = acc[gg][d];
  }
  named_sync(kBarNamedCons, kMkConsThreads);
  for (int i = tid; i < G * D; i += kMkConsThreads) {
    const int gg = i / D, d = i % D;
    float M = -INFINITY;
    for (int w = 0; w < kMkCons; ++w) M = fmaxf(M, wm[w * G + gg]);
    float L = 0.0f, A = 0.0f;
    if (M != -INFINITY)
      for (int w = 0; w < kMkCons; ++w) {
        const float f = __expf(wm[w * G + gg] - M);
        L += wl[w * G + gg] * f;
        A += wacc[(w * G + gg) * D + d] * f;
      }
    const int hq = hk * G + gg;
    if (active == 1) {
      P.o[size_t(hq) * D + d] = L > 0.0f ? __fdividef(A, L) : 0.0f;
    } else {
      const size_t idx = size_t(hq) * P.nsplit_max + sp;
      P.part_o[idx * D + d] = A;
      if (d == 0) {
        P.part_ml[idx * 2] = M;
        P.part_ml[idx * 2 + 1] = L;
      }
    }
  }
  if (active == 1) return;
  __threadfence();
  named_sync(kBarNamedCons, kMkConsThreads);
  if (tid == 0) {
    const int done = atomicAdd(&P.attn_cnt[hk], 1);
    sh.attn_last = done == active - 1;
    if (sh.attn_last) P.attn_cnt[hk] = 0;
  }
  named_sync(kBarNamedCons, kMkConsThreads);
  if (!sh.attn_last) return;
  __threadfence();
  for (int i = tid; i < G * D; i += kMkConsThreads) {
    const int gg = i / D, d = i % D;
    const size_t base = size_t(hk * G + gg) * P.nsplit_max;
    float M = -INFINITY;
    for (int s2 = 0; s2 < active; ++s2) M = fmaxf(M, __ldcg(&P.part_ml[(base + s2) * 2]));
    float L = 0.0f, A = 0.0f;
    for (int s2 = 0; s2 < active; ++s2) {
      const float ms = __ldcg(&P.part_ml[(base + s2) * 2]);
      if (ms == -INFINITY) continue;
      const float f = __expf(ms - M);
      L += __ldcg(&P.part_ml[(base + s2) * 2 + 1]) * f;
      A += __ldcg(&P.part_o[(base + s2) * D + d]) * f;
    }
    P.o[size_t(hk * G + gg) * D + d] = L > 0.0f ? __fdividef(A, L) : 0.0f;
  }
}

// ------------------------------------------------------------------ kernel
template <int FMT, int D, int G>
__global__ void __launch_bounds__(kMkThreads, 1) decode_mk_kernel(const MkParams P) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ MkShared sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* xs = smem;
  uint8_t* scs = smem + P.xs_bytes;                 // 2 scale slots
  uint8_t* ring = scs + 2 * size_t(P.sc_bytes);     // n_slots x 32 KB
  const int L = P.n_layers;
  const int n_bar = 2 + 5 * L;                      // embed, 5 per layer, head

  if (threadIdx.x == 0) {
    for (int s = 0; s < P.n_slots; ++s) {
      mbar_init(&sh.full[s], 1);
      mbar_init(&sh.empty[s], kMkCons);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sh.sc_full[b], 1);
      mbar_init(&sh.sc_empty[b], 1);
      mbar_init(&sh.tile_full[b], kMkCons);
      mbar_init(&sh.tile_free[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    sh.target_base = unsigned(*P.epoch) * unsigned(n_bar) * gridDim.x;
    sh.tok = *P.tok;
    sh.pos = *P.pos;
    sh.slot = *P.slot;
    sh.step = *P.step;
  }
  __syncthreads();

  // ------------------------------------------------------------- producer
  if (warp == kMkCons) {
    if (lane != 0) return;
    int slot = 0, qs = 0;
    uint32_t phase = 0;
    auto stream = [&](const MkLinear& Lw, int fmt) {
      const Slice sl = make_slice(Lw, fmt);
      if (sl.nt == 0) return;
      const int sb = scale_bytes(Lw, fmt, sl);
      if (sb > 0) {
        const int b = qs & 1;
        mbar_wait(&sh.sc_empty[b], ((qs >> 1) & 1) ^ 1);
        mbar_expect_tx(&sh.sc_full[b], sb);
        const size_t row_bytes = fmt == kW4 ? size_t(Lw.k / kW4Group) * 2 : 4;
        bulk_g2s(scs + size_t(b) * P.sc_bytes,
                 static_cast<const uint8_t*>(Lw.s) + size_t(sl.tb) * 16 * row_bytes, sb, &sh.sc_full[b]);
        ++qs;
      }
      const uint8_t* src = static_cast<const uint8_t*>(Lw.w_tf) + size_t(sl.tb) * sl.ct * 512;
      for (int st = 0; st < sl.stages; ++st) {
        const int bytes = min(sl.S, sl.total - st * sl.S) * 512;
        mbar_wait(&sh.empty[slot], phase ^ 1);
        mbar_expect_tx(&sh.full[slot], bytes);
        bulk_g2s(ring + size_t(slot) * kMkSlotBytes, src + size_t(st) * sl.S * 512, bytes, &sh.full[slot]);
        if (++slot == P.n_slots) {
          slot = 0;
          phase ^= 1;
        }
      }
    };
    for (int l = 0; l < L; ++l) {
      const MkLayer& Ly = P.layers[l];
      stream(Ly.qkv, FMT);
      stream(Ly.o, FMT);
      stream(Ly.gu, FMT);
      stream(Ly.down, FMT);
    }
    stream(P.head, kFP16);
    return;
  }

  // ------------------------------------------------------------- epilogue
  if (warp == kMkCons + 1) {
    int tile_ctr = 0, qs = 0;
    unsigned long long best = 0;
    auto phase_epi = [&](const MkLinear& Lw, int fmt, int epi, float* y, bool head) {
      const Slice sl = make_slice(Lw, fmt);
      named_sync(kBarNamedHand, kMkConsThreads + 32);  // consumers passed the input barrier + prologue
      if (sl.nt > 0) {
        const int sb = scale_bytes(Lw, fmt, sl);
        const uint8_t* sc = scs + size_t(qs & 1) * P.sc_bytes;
        if (sb > 0) mbar_wait(&sh.sc_full[qs & 1], (qs >> 1) & 1);
        if (fmt == kINT8) {
          if (epi == kMkResid) mk_epilogue<kINT8, kMkResid>(sl, Lw, sc, y, tile_ctr, sh, best);
          else if (epi == kMkSwiglu) mk_epilogue<kINT8, kMkSwiglu>(sl, Lw, sc, y, tile_ctr, sh, best);
          else mk_epilogue<kINT8, kMkStore>(sl, Lw, sc, y, tile_ctr, sh, best);
        } else {
          if (head) mk_epilogue<kFP16, kMkHead>(sl, Lw, sc, y, tile_ctr, sh, best);
          else if (epi == kMkResid) mk_epilogue<kFP16, kMkResid>(sl, Lw, sc, y, tile_ctr, sh, best);
          else if (epi == kMkSwiglu) mk_epilogue<kFP16, kMkSwiglu>(sl, Lw, sc, y, tile_ctr, sh, best);
          else mk_epilogue<kFP16, kMkStore>(sl, Lw, sc, y, tile_ctr, sh, best);
        }
        if (sb > 0) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&sh.sc_empty[qs & 1]);
          ++qs;
        }
      }
      if (head) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const unsigned long long ob = __shfl_xor_sync(0xffffffffu, best, o);
          best = ob > best ? ob : best;
        }
        if (lane == 0 && best != 0) atomicMax(P.amax, best);
      }
      __syncwarp();
      if (lane == 0) grid_arrive(P);
    };
    for (int l = 0; l < L; ++l) {
      const MkLayer& Ly = P.layers[l];
      phase_epi(Ly.qkv, FMT, kMkStore, P.qkv, false);
      phase_epi(Ly.o, FMT, kMkResid, P.h, false);
      phase_epi(Ly.gu, FMT, kMkSwiglu, P.act, false);
      phase_epi(Ly.down, FMT, kMkResid, P.h, false);
    }
    phase_epi(P.head, kFP16, kMkHead, P.logits, true);
    return;
  }

  // ------------------------------------------------------------- consumers
  const int tid = threadIdx.x;
  int slot = 0, qs = 0, tile_ctr = 0;
  uint32_t phase = 0;
  int bar_j = 0;
  // embedding: h = embed[tok] (fp32), each CTA a slice
  {
    const int per = (P.H + gridDim.x - 1) / gridDim.x;
    const int i0 = blockIdx.x * per, i1 = min(P.H, i0 + per);
    const half* er = P.embed + size_t(sh.tok) * P.H;
    for (int i = i0 + tid; i < i1; i += kMkConsThreads) P.h[i] = __half2float(er[i]);
    named_sync(kBarNamedCons, kMkConsThreads);
    if (tid == 0) grid_arrive(P);
  }
  auto gemv = [&](const MkLinear& Lw, int fmt, const float* x, const half* gamma) {
    const Slice sl = make_slice(Lw, fmt);
    if (tid == 0) grid_wait(P, sh, bar_j);
    named_sync(kBarNamedCons, kMkConsThreads);
    ++bar_j;
    if (sl.nt > 0) {
      if (fmt == kINT8) {
        if (gamma) mk_prologue<kINT8, true>(x, gamma, P.eps, Lw.k, xs, sh);
        else mk_prologue<kINT8, false>(x, gamma, P.eps, Lw.k, xs, sh);
      } else if (fmt == kW4) {
        if (gamma) mk_prologue<kW4, true>(x, gamma, P.eps, Lw.k, xs, sh);
        else mk_prologue<kW4, false>(x, gamma, P.eps, Lw.k, xs, sh);
      } else {
        if (gamma) mk_prologue<kFP16, true>(x, gamma, P.eps, Lw.k, xs, sh);
        else mk_prologue<kFP16, false>(x, gamma, P.eps, Lw.k, xs, sh);
      }
    }
    named_sync(kBarNamedHand, kMkConsThreads + 32);  // hand-off to the epilogue warp
    if (sl.nt == 0) return;
    const int sb = scale_bytes(Lw, fmt, sl);
    const half* sc_h = reinterpret_cast<const half*>(scs + size_t(qs & 1) * P.sc_bytes);
    if (sb > 0) {
      if (fmt == kW4) mbar_wait(&sh.sc_full[qs & 1], (qs >> 1) & 1);
      ++qs;
    }
    const int groups_k = Lw.k / kW4Group;
    if (fmt == kW4) {
      if (sl.ct == kMkMaxS)
        mk_consume<kW4, true>(sl, groups_k, xs, ring, sc_h, P.n_slots, slot, phase, tile_ctr, sh, P.one);
      else
        mk_consume<kW4, false>(sl, groups_k, xs, ring, sc_h, P.n_slots, slot, phase, tile_ctr, sh, P.one);
    } else if (fmt == kINT8) {
      mk_consume<kINT8, false>(sl, groups_k, xs, ring, sc_h, P.n_slots, slot, phase, tile_ctr, sh, P.one);
    } else {
      mk_consume<kFP16, false>(sl, groups_k, xs, ring, sc_h, P.n_slots, slot, phase, tile_ctr, sh, P.one);
    }
  };
  for (int l = 0; l < L; ++l) {
    const MkLayer& Ly = P.layers[l];
    gemv(Ly.qkv, FMT, P.h, Ly.attn_norm);
    // attention (input: qkv of this layer)
    if (tid == 0) grid_wait(P, sh, bar_j);
    named_sync(kBarNamedCons, kMkConsThreads);
    ++bar_j;
    mk_attention<D, G>(P, Ly, xs, sh);
    named_sync(kBarNamedCons, kMkConsThreads);
    if (tid == 0) grid_arrive(P);
    gemv(Ly.o, FMT, P.o, nullptr);
    gemv(Ly.gu, FMT, P.h, Ly.ffn_norm);
    gemv(Ly.down, FMT, P.act, nullptr);
  }
  gemv(P.head, kFP16, P.h, P.final_norm);
  // final: CTA 0 publishes the greedy token and advances the decode state
  if (blockIdx.x == 0 && tid == 0) {
    grid_wait(P, sh, bar_j);
    const unsigned long long k = atomicExch(P.amax, 0ull);
    const int next = int(0xFFFFFFFFu - uint32_t(k & 0xFFFFFFFFull));
    P.next[0] = next;
    P.hist[sh.step] = next;
    *P.tok = next;
    *P.step = sh.step + 1;
    const int p = sh.pos + 1;
    *P.pos = p;
    *P.slot = P.block_table[p >> 4] * 16 + (p & 15);
    *P.epoch = *P.epoch + 1;
  }
}

template <int FMT, int D, int G>
void launch_mk_t(const MkParams& P, size_t smem, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    MSW_CUDA(cudaFuncSetAttribute(decode_mk_kernel<FMT, D, G>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, int(kMkSmemMax)));
    cudaFuncAttributes fa{};
    MSW_CUDA(cudaFuncGetAttributes(&fa, decode_mk_kernel<FMT, D, G>));
    if (fa.maxThreadsPerBlock < kMkThreads || size_t(fa.maxDynamicSharedSizeBytes) < smem)
      throw ConfigErr("decode step kernel resources: maxThreadsPerBlock " +
                      std::to_string(fa.maxThreadsPerBlock) + ", regs " + std::to_string(fa.numRegs) +
                      ", static smem " + std::to_string(fa.sharedSizeBytes) + ", local " +
                      std::to_string(fa.localSizeBytes) + ", max dyn smem " +
                      std::to_string(fa.maxDynamicSharedSizeBytes) + ", requested " + std::to_string(smem));
    attr = true;
  }
  decode_mk_kernel<FMT, D, G><<<kNumSMs, kMkThreads, smem, st>>>(P);
  MSW_LAUNCH_CHECK();
}

template <int FMT>
void launch_mk_fmt(const MkParams& P, size_t smem, cudaStream_t st) {
  const int G = P.Hq / P.Hk;
#define MSW_MK(DD, GG) \
  if (P.D == DD && G == GG) return launch_mk_t<FMT, DD, GG>(P, smem, st);
  MSW_MK(128, 4)
  MSW_MK(64, 4)
  MSW_MK(128, 2)
  MSW_MK(64, 2)
  MSW_MK(128, 1)
  MSW_MK(64, 1)
#undef MSW_MK
  throw ConfigErr("decode step: unsupported head_dim / GQA group");
}

}  // namespace

size_t mk_smem_plan(MkParams& P, int fmt) {
  auto xs_need = [&](int k) -> size_t {
    return fmt == kINT8 ? size_t(k) : size_t(2) * k + size_t(4) * (k / kW4Group);
  };
  const int G = P.Hq / P.Hk;
  size_t xs = std::max({xs_need(P.H), xs_need(P.Hq * P.D), xs_need(P.F), size_t(2) * P.H});
  const size_t attn = size_t(G) * P.D * 4 + size_t(2) * P.D * 2 + size_t(2) * kMkCons * G * 4 +
                      size_t(kMkCons) * G * P.D * 4;
  xs = std::max(xs, attn);
  xs = (xs + 127) & ~size_t(127);
  size_t sc = 0;
  auto sc_need = [&](int n, int k) -> size_t {
    const int ntiles = n / 16;
    const int per = (ntiles + kNumSMs - 1) / kNumSMs;
    return fmt == kW4 ? size_t(per) * 16 * (k / kW4Group) * 2 : (fmt == kINT8 ? size_t(per) * 16 * 4 : 0);
  };
  sc = std::max({sc_need((P.Hq + 2 * P.Hk) * P.D, P.H), sc_need(P.H, P.Hq * P.D),
                 sc_need(2 * P.F, P.H), sc_need(P.H, P.F)});
  sc = (sc + 127) & ~size_t(127);
  const size_t fixed = xs + 2 * sc;
  if (fixed + 2 * size_t(kMkSlotBytes) > kMkSmemMax) throw ConfigErr("decode step: shared memory budget");
  const int slots = int(std::min<size_t>(kMkMaxSlots, (kMkSmemMax - fixed) / kMkSlotBytes));
  P.xs_bytes = int(xs);
  P.sc_bytes = int(sc);
  P.n_slots = slots;
  return fixed + size_t(slots) * kMkSlotBytes;
}

bool mk_supported(const MkParams& P) {
  auto ok = [](int k) { return k % 128 == 0 && k <= kMkXRegs * 4 * kMkConsThreads; };
  const int G = P.Hk > 0 ? P.Hq / P.Hk : 0;
  return ok(P.H) && ok(P.Hq * P.D) && ok(P.F) && (P.D == 64 || P.D == 128) &&
         (G == 1 || G == 2 || G == 4) && P.Hq % P.Hk == 0;
}

void launch_decode_mk(int fmt, const MkParams& P, size_t smem, cudaStream_t st) {
  switch (fmt) {
    case kFP16: return launch_mk_fmt<kFP16>(P, smem, st);
    case kINT8: return launch_mk_fmt<kINT8>(P, smem, st);
    case kW4: return launch_mk_fmt<kW4>(P, smem, st);
    default: throw ConfigErr("decode step: bad format");
  }
}

}  // namespace msw
