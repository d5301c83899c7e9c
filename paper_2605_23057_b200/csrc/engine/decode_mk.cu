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
// (gemv.cu, attention.cu, misc.cu); W4 uses gemv.cu's single-lop3 dequant
// ((1024 + q) against x on even k16 steps, (1024 + 16 q) against x/16 on odd
// ones, per-group offset removed before the group scale).
#include <algorithm>
#include <type_traits>

#include "kernels.cuh"
#include "mma_frag.cuh"

namespace msw {
#ifdef MSW_TRACE
__device__ unsigned long long* g_mk_trace = nullptr;
extern "C" int msw_mk_trace_set(void* buf) {
  return cudaMemcpyToSymbol(g_mk_trace, &buf, sizeof(buf)) == cudaSuccess ? 0 : 1;
}
// globaltimer (ns) at event e of CTA b: buf[b * 8192 + e]
//   0..299 consumer past barrier j, 300..599 epilogue arrival, 600..899 producer
//   phase start, 900.. attention done, 1000 embed; 1024+s producer issued stage s,
//   2048+s consumer warp 0 got stage s, 3072+t epilogue finished tile t,
//   4096+j prologue of the GEMV phase after barrier j done
#define MK_TP(e)                                                      \
  do {                                                                \
    if (g_mk_trace) {                                                 \
      unsigned long long g_;                                          \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_));          \
      g_mk_trace[blockIdx.x * 8192 + (e)] = g_;                       \
    }                                                                 \
  } while (0)
#else
#define MK_TP(e) \
  do {           \
  } while (0)
#endif
namespace {

constexpr int kMkCons = 16;
constexpr int kMkThreads = (kMkCons + 2) * 32;
constexpr int kMkConsThreads = kMkCons * 32;
constexpr int kMkCPW = 4;                       // chunks per warp per stage
constexpr int kMkMaxS = kMkCons * kMkCPW;       // 64 chunks of 512 B
constexpr int kMkSlotBytes = kMkMaxS * 512;     // 32 KB ring slot
constexpr int kMkMaxSlots = 8;
constexpr int kMkXRegs = 4;                     // float4 of x kept per thread (k <= 8192)
constexpr int kMkAttnMinChunk = 128;            // positions per attention split, at least
constexpr int kBarNamedCons = 1;                // named barrier: consumers
constexpr int kBarNamedHand = 3;                // named barrier: consumers + epilogue

enum MkEpi { kMkStore = 0, kMkResid = 1, kMkSwiglu = 2, kMkHead = 3 };

__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
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
  uint64_t kv_full[2];
  uint32_t kv_par[2];  // parity of the next completion of kv_full[b] (carried across layers)
  float part[2][kMkCons][16];
  float red[32];
  float xscale;
  int attn_last;
  unsigned target_base;
  int tok, pos, slot, step;
  int trace_cs, trace_et, trace_pro;  // diagnostics counters (MSW_TRACE builds)
};

// Ring / tile-buffer position of the consumer warps, passed and returned BY
// VALUE: with ~28 KB of L1 left beside the 223 KB smem carve-out, anything
// in local memory (references to caller locals, spills) costs an L2 round
// trip, so the hot loops must keep all state in registers.
struct RingState {
  int slot;
  uint32_t phase;
  int tile_ctr;
};
struct EpiState {
  int tile_ctr;
  unsigned long long best;
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
// The arriving thread follows a __syncwarp / named barrier over the threads
// whose writes it publishes; red.release.gpu is cumulative over those.
__device__ __forceinline__ void grid_arrive(const MkParams& P) { red_release_add(P.bar, 1u); }
// Polls with relaxed loads (an ld.acquire per poll compiles to a full L1
// invalidate, CCTL.IVALL, each iteration) and acquires once with a fence.
__device__ __forceinline__ void grid_wait(const MkParams& P, const MkShared& sh, int j) {
  const unsigned target = sh.target_base + unsigned(j + 1) * gridDim.x;
  while (int(ld_relaxed_u32(P.bar) - target) < 0) {
  }
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// o[4i .. 4i+3] (one head's dims) from the attention partials of `active` splits
__device__ __forceinline__ float4 attn_merge4(const MkParams& P, int active, int i) {
  const int e = 4 * i, hq = e / P.D, d = e % P.D;
  const size_t base = size_t(hq) * P.nsplit_max;
  const float2* ml = reinterpret_cast<const float2*>(P.part_ml) + base;
  const float* po = P.part_o + base * P.D + d;
  if (active == 1) {  // one split: o = A / L
    const float2 m = __ldcg(ml);
    const float4 a = __ldcg(reinterpret_cast<const float4*>(po));
    const float inv = m.y > 0.0f ? 1.0f / m.y : 0.0f;
    return make_float4(a.x * inv, a.y * inv, a.z * inv, a.w * inv);
  }
  float Mx = -INFINITY;
  for (int s2 = 0; s2 < active; ++s2) Mx = fmaxf(Mx, __ldcg(ml + s2).x);
  float Ls = 0.0f;
  float4 As = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int s2 = 0; s2 < active; ++s2) {
    const float2 m = __ldcg(ml + s2);
    if (m.x == -INFINITY) continue;
    const float4 a = __ldcg(reinterpret_cast<const float4*>(po + size_t(s2) * P.D));
    const float f = __expf(m.x - Mx);
    Ls += m.y * f;
    As.x += a.x * f;
    As.y += a.y * f;
    As.z += a.z * f;
    As.w += a.w * f;
  }
  if (!(Ls > 0.0f)) return make_float4(0.f, 0.f, 0.f, 0.f);
  const float inv = 1.0f / Ls;
  return make_float4(As.x * inv, As.y * inv, As.z * inv, As.w * inv);
}

// --------------------------------------------------------------- prologue
// x fp32 [k] (global, written by earlier phases) -> xs (smem):
//   FP16: fp16 [k] permuted (perm_f16); INT8: int8 [k] permuted (perm_i8) +
//   sh.xscale; W4: fp16 [k] permuted + float corr[k/128] = 1032 * sum(x | even k16
//   steps of the group) + 72 * sum(x | odd steps).
// Thread t handles float4 i = t + 512 j (registers between the passes); warp w
// covers k in [128 (w + 16 j), +128) = one W4 scale group per j.
template <int FMT, bool NORM, bool ATTN>
__device__ __noinline__ void mk_prologue(const float* __restrict__ x,
                                         const half* __restrict__ gamma, float eps, int k,
                                         uint8_t* xs, MkShared& sh, const MkParams* attn,
                                         int attn_active) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k4 = k >> 2;
  const float4* xt = reinterpret_cast<const float4*>(x);
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
#ifdef MSW_TRACE
  const int tp = sh.trace_pro;
  if (tid == 0) MK_TP(5000 + 5 * tp);
#endif
  auto load = [&](int j) -> float4 {
    const int i = tid + j * kMkConsThreads;
    if constexpr (ATTN) return attn_merge4(*attn, attn_active, i);
    else return __ldcg(xt + i);
  };
  // Every load of the phase input (x, gamma) is issued up front: one L2 round
  // trip (~1 us under the weight stream) instead of one per pass.
  constexpr int NREG = ATTN ? 2 : (NORM ? 4 : 8);  // float4 per thread: k <= 4096 / 8192 / 16384
  const bool in_regs = k4 <= NREG * kMkConsThreads;
  float4 v[NREG];
  uint2 gv[NORM ? NREG : 1];
  if (in_regs) {
#pragma unroll
    for (int j = 0; j < NREG; ++j)
      if (tid + j * kMkConsThreads < k4) {
        v[j] = load(j);
        if (NORM) gv[NORM ? j : 0] = reinterpret_cast<const uint2*>(gamma)[tid + j * kMkConsThreads];
      }
  }
  auto get = [&](int j) -> float4 { return in_regs ? v[j] : load(j); };
  auto gam = [&](int j) -> uint2 {
    return in_regs ? gv[NORM ? j : 0] : reinterpret_cast<const uint2*>(gamma)[tid + j * kMkConsThreads];
  };
  float r = 1.0f;
  if (NORM) {
    float ss = 0.0f;
#pragma unroll 4
    for (int j = 0; j * kMkConsThreads < k4; ++j)
      if (tid + j * kMkConsThreads < k4) {
        const float4 a = get(j);
        ss = fmaf(a.x, a.x, fmaf(a.y, a.y, fmaf(a.z, a.z, fmaf(a.w, a.w, ss))));
      }
#ifdef MSW_TRACE
    if (tid == 0) MK_TP(5000 + 5 * tp + 1);  // x arrived (first use)
#endif
    ss = sync_red(ss, false);
#ifdef MSW_TRACE
    if (tid == 0) MK_TP(5000 + 5 * tp + 2);  // reduction done
#endif
    r = 1.0f / sqrtf(ss / float(k) + eps);
  }
  auto act = [&](int j) -> float4 {
    float4 a = get(j);
    if (NORM) {
      const uint2 gg = gam(j);
      const float2 g0 = __half22float2(*reinterpret_cast<const half2*>(&gg.x));
      const float2 g1 = __half22float2(*reinterpret_cast<const half2*>(&gg.y));
      a.x = (a.x * r) * g0.x;
      a.y = (a.y * r) * g0.y;
      a.z = (a.z * r) * g1.x;
      a.w = (a.w * r) * g1.y;
    }
    return a;
  };
  if (FMT == kINT8) {
    float amax = 0.0f;
#pragma unroll 4
    for (int j = 0; j * kMkConsThreads < k4; ++j)
      if (tid + j * kMkConsThreads < k4) {
        const float4 a = act(j);
        amax = fmaxf(amax, fmaxf(fmaxf(fabsf(a.x), fabsf(a.y)), fmaxf(fabsf(a.z), fabsf(a.w))));
      }
    amax = sync_red(amax, true);
    const float s = amax / 127.0f;
    auto q = [&](float val) -> int8_t {
      const float u = amax > 0.0f ? rintf(val / s) : 0.0f;
      return static_cast<int8_t>(fminf(fmaxf(u, -127.0f), 127.0f));
    };
    int8_t* xq = reinterpret_cast<int8_t*>(xs);
#pragma unroll 4
    for (int j = 0; j * kMkConsThreads < k4; ++j) {
      const int i = tid + j * kMkConsThreads;
      if (i < k4) {
        const float4 a = act(j);
        *reinterpret_cast<char4*>(xq + perm_i8(4 * i)) = make_char4(q(a.x), q(a.y), q(a.z), q(a.w));
      }
    }
    if (tid == 0) sh.xscale = s;
  } else {
    half* xh = reinterpret_cast<half*>(xs);
    float* corr = reinterpret_cast<float*>(xs + size_t(2) * k);
#pragma unroll 4
    for (int j = 0; j * kMkConsThreads < k4; ++j) {
      const int i = tid + j * kMkConsThreads;
      if (warp * 32 + j * kMkConsThreads >= k4) continue;  // warp-uniform (k4 % 32 == 0)
      const float4 a = act(j);
      const half2 lo = __floats2half2_rn(a.x, a.y), hi = __floats2half2_rn(a.z, a.w);
      *reinterpret_cast<half2*>(xh + perm_f16(4 * i)) = lo;
      *reinterpret_cast<half2*>(xh + perm_f16(4 * i + 2)) = hi;
      if (FMT == kW4) {  // lane bit 2 = k16-step parity: even sums in lane 0, odd in lane 4
        const float2 lf = __half22float2(lo), hf = __half22float2(hi);
        float gs = (lf.x + lf.y) + (hf.x + hf.y);
        gs += __shfl_xor_sync(0xffffffffu, gs, 1);
        gs += __shfl_xor_sync(0xffffffffu, gs, 2);
        gs += __shfl_xor_sync(0xffffffffu, gs, 8);
        gs += __shfl_xor_sync(0xffffffffu, gs, 16);
        const float odd = __shfl_sync(0xffffffffu, gs, 4);
        if (lane == 0) corr[warp + j * kMkCons] = 1032.0f * gs + 72.0f * odd;
      }
    }
  }
#ifdef MSW_TRACE
  if (tid == 0) MK_TP(5000 + 5 * tp + 3);  // converted
#endif
  named_sync(kBarNamedCons, kMkConsThreads);
#ifdef MSW_TRACE
  if (tid == 0) {
    MK_TP(5000 + 5 * tp + 4);
    ++sh.trace_pro;
  }
#endif
}

// fp16 pair x -> x / 16 (exact power-of-two scaling), for the odd k16 steps
__device__ __forceinline__ uint2 x16(uint2 b) {
  const half2 s = __float2half2_rn(0.0625f);
  return make_uint2(h22u(__hmul2(u2h2(b.x), s)), h22u(__hmul2(u2h2(b.y), s)));
}

// ------------------------------------------------------------ GEMV consumer
// One linear's share of this CTA: stages of S chunks from the ring; warp w
// takes chunks [4w, 4w + 4) of each stage. Every consumer warp flushes every
// tile exactly once, in order (zero partial if it never touched it).
template <int FMT, bool XREG>
__device__ __noinline__ RingState mk_consume(const Slice sl, int groups_k, const uint8_t* xs,
                                             const uint8_t* ring, const half* sc_h, int n_slots,
                                             RingState rs, MkShared& sh) {
  int slot = rs.slot, tile_ctr = rs.tile_ctr;
  uint32_t phase = rs.phase;
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
        bx[XREG ? j : 0][p][1] = x16(*reinterpret_cast<const uint2*>(xrow + kb + 32));
      }
    cx[0] = corr[w0c / 2];
    cx[XREG ? 1 : 0] = corr[w0c / 2 + 1];
  }
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
    mbar_arrive(&sh.tile_full[b]);  // per-lane release of its own stores
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
#ifdef MSW_TRACE
    if (warp == 0 && lane == 0) {
      if (sh.trace_cs < 1024) MK_TP(2048 + sh.trace_cs);
      ++sh.trace_cs;
    }
#endif
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
              // even step 2p: nibbles 0/4 (row g), 2/6 (row g+8) as 1024 + q against x;
              // odd step 2p+1: nibbles 1/5, 3/7 as 1024 + 16 q against x/16 (one SHF
              // per word serves four lop3s; IMAD.HI shifts measured ~3x slower)
              const uint32_t w0s = w0 >> 8, w1s = w1 >> 8;
              const uint32_t a_lo[4] = {lop3_and_or(w0, 0x000F000Fu, 0x64006400u),
                                        lop3_and_or(w0s, 0x000F000Fu, 0x64006400u),
                                        lop3_and_or(w1, 0x000F000Fu, 0x64006400u),
                                        lop3_and_or(w1s, 0x000F000Fu, 0x64006400u)};
              const uint32_t a_hi[4] = {lop3_and_or(w0, 0x00F000F0u, 0x64006400u),
                                        lop3_and_or(w0s, 0x00F000F0u, 0x64006400u),
                                        lop3_and_or(w1, 0x00F000F0u, 0x64006400u),
                                        lop3_and_or(w1s, 0x00F000F0u, 0x64006400u)};
              uint2 be, bo;
              if (XREG) {
                be = bx[XREG ? j : 0][p][0];
                bo = bx[XREG ? j : 0][p][1];
              } else {
                const int kb = ((cs + j) * 64 + p * 32) * 2;
                be = *reinterpret_cast<const uint2*>(xrow + kb);
                bo = x16(*reinterpret_cast<const uint2*>(xrow + kb + 32));
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
  return RingState{slot, phase, tile_ctr};
}

// ---------------------------------------------------------- GEMV epilogue
template <int FMT, int EPI>
__device__ __noinline__ EpiState mk_epilogue(const Slice sl, const uint8_t* sc, float* y,
                                             EpiState es, MkShared& sh) {
  const int lane = threadIdx.x & 31;
  int tile_ctr = es.tile_ctr;
  unsigned long long best = es.best;
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
#ifdef MSW_TRACE
    if (lane == 0) {
      if (sh.trace_et < 1024) MK_TP(3072 + sh.trace_et);
      ++sh.trace_et;
    }
#endif
    ++tile_ctr;
  }
  return EpiState{tile_ctr, best};
}

// -------------------------------------------------------------- attention
// Decode attention of one layer for the single new token at position p.
// Work item (kv head hk, split sp) = CTA blockIdx.x; the split covers
// positions [begin, end) in 32-position sub-chunks. The cached K/V of a
// sub-chunk are two 16-position paged blocks per head, each 16 x D fp16
// contiguous, so they arrive as cp.async.bulk copies into shared memory
// (double-buffered); the first two are issued BEFORE the phase barrier (the
// history is immutable), hiding the load latency behind the QKV phase.
// Per sub-chunk: QK with warps over positions and lanes over D (shuffle
// reduce), then every consumer thread owns one (head, dim) output and runs
// the online softmax + PV over the sub-chunk from shared memory. Across
// splits, the last CTA of a head (counter) merges the (m, l, acc) partials.
// Numerics as attention.cu: fp16 q/k/v after RoPE, fp32 scores / softmax /
// accumulation, scale 1/sqrt(D).
constexpr int kMkSub = 32;  // positions per sub-chunk (two KV blocks)

struct AttnWork {
  int active, hk, sp, begin, end, nsub;
};
__device__ __forceinline__ AttnWork attn_work(const MkParams& P, int pos) {
  AttnWork w{};
  const int ctx = pos + 1;
  int nsplit = min(P.nsplit_max, max(1, int(gridDim.x) / P.Hk));
  nsplit = min(nsplit, max(1, (ctx + kMkAttnMinChunk - 1) / kMkAttnMinChunk));
  int chunk = (ctx + nsplit - 1) / nsplit;
  chunk = ((chunk + kMkSub - 1) / kMkSub) * kMkSub;
  w.active = (ctx + chunk - 1) / chunk;
  const int item = blockIdx.x;
  if (item >= P.Hk * w.active) {
    w.nsub = 0;
    return w;
  }
  w.hk = item % P.Hk;
  w.sp = item / P.Hk;
  w.begin = w.sp * chunk;
  w.end = min(ctx, w.begin + chunk);
  w.nsub = (w.end - w.begin + kMkSub - 1) / kMkSub;
  return w;
}

template <int D>
__device__ __forceinline__ size_t attn_kv_bytes() { return size_t(2) * kMkSub * D * 2; }  // K + V

// Issues the bulk copies of sub-chunk i (K and V of its <= 2 blocks) into
// buffer (i & 1). Called by one thread.
template <int D>
__device__ __forceinline__ void attn_issue(const MkParams& P, const MkLayer& Ly, const AttnWork& w,
                                           int i, uint8_t* xs, MkShared& sh) {
  uint8_t* buf = xs + (i & 1) * attn_kv_bytes<D>();
  const int p0 = w.begin + i * kMkSub;
  const int nblk = min(2, (min(w.end, p0 + kMkSub) - p0 + 15) / 16);
  const uint32_t blk_bytes = 16 * D * 2;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // after generic reads of buf
  mbar_expect_tx(&sh.kv_full[i & 1], 2 * nblk * blk_bytes);
  for (int b = 0; b < nblk; ++b) {
    const int blk = P.block_table[(p0 >> 4) + b];
    const size_t off = (size_t(blk) * P.Hk + w.hk) * 16 * D;
    bulk_g2s(buf + b * blk_bytes, Ly.kc + off, blk_bytes, &sh.kv_full[i & 1]);
    bulk_g2s(buf + kMkSub * D * 2 + b * blk_bytes, Ly.vc + off, blk_bytes, &sh.kv_full[i & 1]);
  }
}

// Before the attention barrier (thread 0, after the consumers are done with xs).
template <int D>
__device__ __forceinline__ void mk_attn_prefetch(const MkParams& P, const MkLayer& Ly,
                                                 uint8_t* xs, MkShared& sh) {
  const AttnWork w = attn_work(P, sh.pos);
  for (int i = 0; i < min(2, w.nsub); ++i) attn_issue<D>(P, Ly, w, i, xs, sh);
}

template <int D, int G>
__device__ __noinline__ void mk_attention(const MkParams& P, const MkLayer& Ly, uint8_t* xs,
                                          MkShared& sh) {
  static_assert(G * D <= kMkConsThreads, "one (head, dim) output per consumer thread");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int Hq = P.Hq, Hk = P.Hk;
  const int p_self = sh.pos;
  const AttnWork w = attn_work(P, p_self);
  if (w.nsub == 0) return;
  const int hk = w.hk;
  // smem: [2 buffers: K 32xD | V 32xD] | qs[G][D] f32 | knew[D], vnew[D] f16 | sc[G][32]
  half* kvb = reinterpret_cast<half*>(xs);
  float* qs = reinterpret_cast<float*>(xs + 2 * attn_kv_bytes<D>());
  half* knew = reinterpret_cast<half*>(qs + G * D);
  half* vnew = knew + D;
  float* scs = reinterpret_cast<float*>(vnew + D);
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
  if (w.sp == 0) {
    const size_t off = ((size_t(sh.slot >> 4) * Hk + hk) * 16 + (sh.slot & 15)) * size_t(D);
    for (int d = tid; d < D; d += kMkConsThreads) {
      Ly.kc[off + d] = knew[d];
      Ly.vc[off + d] = vnew[d];
    }
  }
  const uint32_t par0 = sh.kv_par[0], par1 = sh.kv_par[1];
  const float scale = rsqrtf(float(D));
  // PV ownership: thread -> (g, d)
  const bool owner = tid < G * D;
  const int og = tid / D, od = tid % D;
  float M = -INFINITY, L = 0.0f, A = 0.0f;
  // QK: warp -> 2 positions (lanes 0-15 / 16-31), 16 lanes x D/16 dims
  constexpr int DPL = D / 16;
  const int qp = 2 * warp + (lane >> 4);
  const int ql = lane & 15;
#pragma unroll 1
  for (int i = 0; i < w.nsub; ++i) {
    const int b = i & 1;
    mbar_wait(&sh.kv_full[b], (b ? par1 : par0) ^ ((i >> 1) & 1));
    const half* Kb = kvb + b * (attn_kv_bytes<D>() / 2);
    const half* Vb = Kb + kMkSub * D;
    const int p0 = w.begin + i * kMkSub;
    const int pq = p0 + qp;
    float sg[G];
#pragma unroll
    for (int gg = 0; gg < G; ++gg) sg[gg] = 0.0f;
    {
      const half* kr = pq == p_self ? knew : Kb + qp * D;
#pragma unroll
      for (int c = 0; c < DPL; c += 4) {  // 4 dims per step (D = 64: one step, D = 128: two)
        const uint2 kv = *reinterpret_cast<const uint2*>(kr + ql * DPL + c);
        const float2 k0 = __half22float2(*reinterpret_cast<const half2*>(&kv.x));
        const float2 k1 = __half22float2(*reinterpret_cast<const half2*>(&kv.y));
#pragma unroll
        for (int gg = 0; gg < G; ++gg) {
          const float4 q0 = *reinterpret_cast<const float4*>(qs + gg * D + ql * DPL + c);
          sg[gg] = fmaf(q0.x, k0.x, fmaf(q0.y, k0.y, fmaf(q0.z, k1.x, fmaf(q0.w, k1.y, sg[gg]))));
        }
      }
    }
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) sg[gg] += __shfl_xor_sync(0xffffffffu, sg[gg], o);
      if (ql == 0) scs[gg * kMkSub + qp] = pq < w.end ? sg[gg] * scale : -INFINITY;
    }
    named_sync(kBarNamedCons, kMkConsThreads);
    if (owner) {
      float mx = M;
#pragma unroll 8
      for (int j = 0; j < kMkSub; ++j) mx = fmaxf(mx, scs[og * kMkSub + j]);
      const float corr = __expf(M - mx);
      A *= corr;
      L *= corr;
      M = mx;
#pragma unroll 8
      for (int j = 0; j < kMkSub; ++j) {
        const float sv = scs[og * kMkSub + j];
        if (sv == -INFINITY) continue;  // past the split end: stale buffer contents
        const float e = __expf(sv - mx);
        const half v = (p0 + j) == p_self ? vnew[od] : Vb[j * D + od];
        L += e;
        A = fmaf(e, __half2float(v), A);
      }
    }
    named_sync(kBarNamedCons, kMkConsThreads);  // buffer b and scs are free again
    if (tid == 0 && i + 2 < w.nsub) attn_issue<D>(P, Ly, w, i + 2, xs, sh);
  }
  if (tid == 0) {  // completions this layer: buffer 0 ceil(nsub/2), buffer 1 floor(nsub/2)
    sh.kv_par[0] = par0 ^ (((w.nsub + 1) / 2) & 1);
    sh.kv_par[1] = par1 ^ ((w.nsub / 2) & 1);
  }
  // (m, l, acc) partials; the O-projection prologue merges the splits
  if (owner) {
    const size_t idx = size_t(hk * G + og) * P.nsplit_max + w.sp;
    P.part_o[idx * D + od] = A;
    if (od == 0) {
      P.part_ml[idx * 2] = M;
      P.part_ml[idx * 2 + 1] = L;
    }
  }
}

// ------------------------------------------------------------------ kernel
template <int FMT, int D, int G>
__global__ void __launch_bounds__(kMkThreads, 1) decode_mk_kernel(const __grid_constant__ MkParams P) {
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
      mbar_init(&sh.tile_full[b], kMkCons * 32);
      mbar_init(&sh.tile_free[b], 1);
      mbar_init(&sh.kv_full[b], 1);
      sh.kv_par[b] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    sh.target_base = unsigned(*P.epoch) * unsigned(n_bar) * gridDim.x;
    sh.tok = *P.tok;
    sh.pos = *P.pos;
    sh.slot = *P.slot;
    sh.step = *P.step;
    sh.trace_cs = 0;
    sh.trace_et = 0;
    sh.trace_pro = 0;
#ifdef MSW_TRACE
    if (g_mk_trace) {  // SM clock: clock64 / globaltimer at start (8000) and end (8002)
      unsigned long long g_;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_));
      g_mk_trace[blockIdx.x * 8192 + 8000] = g_;
      g_mk_trace[blockIdx.x * 8192 + 8001] = clock64();
    }
#endif
  }
  __syncthreads();

  // ------------------------------------------------------------- producer
  if (warp == kMkCons) {
    if (lane != 0) return;
    int slot = 0, qs = 0, pq = 0;
    uint32_t phase = 0;
    const uint64_t pol = policy_evict_first();
#ifdef MSW_TRACE
    int gst = 0;
#endif
    auto stream = [&](const MkLinear& Lw, int fmt) {
      const Slice sl = make_slice(Lw, fmt);
      MK_TP(600 + pq);  // producer starts this phase
      ++pq;
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
        bulk_g2s_hint(ring + size_t(slot) * kMkSlotBytes, src + size_t(st) * sl.S * 512, bytes,
                      &sh.full[slot], pol);
#ifdef MSW_TRACE
        if (gst < 1024) MK_TP(1024 + gst);
        ++gst;
#endif
        if (++slot == P.n_slots) {
          slot = 0;
          phase ^= 1;
        }
      }
    };
    const AttnWork aw = attn_work(P, sh.pos);
    for (int l = 0; l < L; ++l) {
      const MkLayer& Ly = P.layers[l];
      // this CTA's attention item of layer l: pull its KV history into L2 now
      // (about a layer ahead of the consumers); the smem copies then hit L2
      for (int p0 = aw.begin; aw.nsub > 0 && p0 < aw.end; p0 += 16) {
        const size_t off = (size_t(P.block_table[p0 >> 4]) * P.Hk + aw.hk) * 16 * D;
        prefetch_l2(Ly.kc + off, 16 * D * 2);
        prefetch_l2(Ly.vc + off, 16 * D * 2);
      }
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
    int qs = 0, eph = 0;
    EpiState es{0, 0ull};
    auto phase_epi = [&](const MkLinear& Lw, int fmt, int epi, float* y, bool head) {
      const Slice sl = make_slice(Lw, fmt);
      named_sync(kBarNamedHand, kMkConsThreads + 32);  // consumers passed the input barrier + prologue
      if (sl.nt > 0) {
        const int sb = scale_bytes(Lw, fmt, sl);
        const uint8_t* sc = scs + size_t(qs & 1) * P.sc_bytes;
        if (sb > 0) mbar_wait(&sh.sc_full[qs & 1], (qs >> 1) & 1);
        if (fmt == kINT8) {
          if (epi == kMkResid) es = mk_epilogue<kINT8, kMkResid>(sl, sc, y, es, sh);
          else if (epi == kMkSwiglu) es = mk_epilogue<kINT8, kMkSwiglu>(sl, sc, y, es, sh);
          else es = mk_epilogue<kINT8, kMkStore>(sl, sc, y, es, sh);
        } else {
          if (head) es = mk_epilogue<kFP16, kMkHead>(sl, sc, y, es, sh);
          else if (epi == kMkResid) es = mk_epilogue<kFP16, kMkResid>(sl, sc, y, es, sh);
          else if (epi == kMkSwiglu) es = mk_epilogue<kFP16, kMkSwiglu>(sl, sc, y, es, sh);
          else es = mk_epilogue<kFP16, kMkStore>(sl, sc, y, es, sh);
        }
        if (sb > 0) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&sh.sc_empty[qs & 1]);
          ++qs;
        }
      }
      if (head) {
        unsigned long long best = es.best;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const unsigned long long ob = __shfl_xor_sync(0xffffffffu, best, o);
          best = ob > best ? ob : best;
        }
        if (lane == 0 && best != 0) atomicMax(P.amax, best);
      }
      __syncwarp();
      if (lane == 0) {
        MK_TP(300 + eph);
        grid_arrive(P);
      }
      ++eph;
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
  int qs = 0;
  RingState rs{0, 0u, 0};
  int bar_j = 0;
  // embedding: h = embed[tok] (fp32), each CTA a slice
  {
    const int per = (P.H + gridDim.x - 1) / gridDim.x;
    const int i0 = blockIdx.x * per, i1 = min(P.H, i0 + per);
    const half* er = P.embed + size_t(sh.tok) * P.H;
    for (int i = i0 + tid; i < i1; i += kMkConsThreads) P.h[i] = __half2float(er[i]);
    named_sync(kBarNamedCons, kMkConsThreads);
    if (tid == 0) {
      MK_TP(1000);  // kernel start (embed done)
      grid_arrive(P);
    }
  }
  const int attn_active = attn_work(P, sh.pos).active;
  auto gemv = [&](const MkLinear& Lw, int fmt, const float* x, const half* gamma,
                  const MkParams* attn) {
    const Slice sl = make_slice(Lw, fmt);
    if (tid == 0) {
      grid_wait(P, sh, bar_j);
      MK_TP(bar_j);
    }
    named_sync(kBarNamedCons, kMkConsThreads);
    ++bar_j;
    if (sl.nt > 0) {
      if (attn) {  // O projection: input = merged attention partials (plain)
        if (fmt == kINT8) mk_prologue<kINT8, false, true>(x, gamma, P.eps, Lw.k, xs, sh, attn, attn_active);
        else if (fmt == kW4) mk_prologue<kW4, false, true>(x, gamma, P.eps, Lw.k, xs, sh, attn, attn_active);
        else mk_prologue<kFP16, false, true>(x, gamma, P.eps, Lw.k, xs, sh, attn, attn_active);
      } else if (fmt == kINT8) {
        if (gamma) mk_prologue<kINT8, true, false>(x, gamma, P.eps, Lw.k, xs, sh, attn, attn_active);
        else mk_prologue<kINT8, false, false>(x, gamma, P.eps, Lw.k, xs, sh, attn, attn_active);
      } else if (fmt == kW4) {
        if (gamma) mk_prologue<kW4, true, false>(x, gamma, P.eps, Lw.k, xs, sh, attn, attn_active);
        else mk_prologue<kW4, false, false>(x, gamma, P.eps, Lw.k, xs, sh, attn, attn_active);
      } else {
        if (gamma) mk_prologue<kFP16, true, false>(x, gamma, P.eps, Lw.k, xs, sh, attn, attn_active);
        else mk_prologue<kFP16, false, false>(x, gamma, P.eps, Lw.k, xs, sh, attn, attn_active);
      }
    }
    named_sync(kBarNamedHand, kMkConsThreads + 32);  // hand-off to the epilogue warp
    if (tid == 0) MK_TP(4096 + bar_j - 1);  // prologue done (phase index = its input barrier)
    if (sl.nt == 0) return;
    const int sb = scale_bytes(Lw, fmt, sl);
    const half* sc_h = reinterpret_cast<const half*>(scs + size_t(qs & 1) * P.sc_bytes);
    if (sb > 0) {
      if (fmt == kW4) mbar_wait(&sh.sc_full[qs & 1], (qs >> 1) & 1);
      ++qs;
    }
    const int groups_k = Lw.k / kW4Group;
    if (fmt == kW4) {
      // (the register-resident XREG variant spills at the 96-register budget of
      // 18 warps/SM; LDS B fragments + HMUL2 for x/16 are cheaper than spills)
      rs = mk_consume<kW4, false>(sl, groups_k, xs, ring, sc_h, P.n_slots, rs, sh);
    } else if (fmt == kINT8) {
      rs = mk_consume<kINT8, false>(sl, groups_k, xs, ring, sc_h, P.n_slots, rs, sh);
    } else {
      rs = mk_consume<kFP16, false>(sl, groups_k, xs, ring, sc_h, P.n_slots, rs, sh);
    }
  };
  for (int l = 0; l < L; ++l) {
    const MkLayer& Ly = P.layers[l];
    gemv(Ly.qkv, FMT, P.h, Ly.attn_norm, nullptr);
    // attention (input: qkv of this layer); its KV history is prefetched first
    named_sync(kBarNamedCons, kMkConsThreads);  // every consumer is done with xs
    if (tid == 0) mk_attn_prefetch<D>(P, Ly, xs, sh);
    if (tid == 0) {
      grid_wait(P, sh, bar_j);
      MK_TP(bar_j);
    }
    named_sync(kBarNamedCons, kMkConsThreads);
    ++bar_j;
    mk_attention<D, G>(P, Ly, xs, sh);
    named_sync(kBarNamedCons, kMkConsThreads);
    if (tid == 0) {
      MK_TP(900 + l);  // attention done
      grid_arrive(P);
    }
    gemv(Ly.o, FMT, nullptr, nullptr, &P);  // input = merged attention partials
    gemv(Ly.gu, FMT, P.h, Ly.ffn_norm, nullptr);
    gemv(Ly.down, FMT, P.act, nullptr, nullptr);
  }
  gemv(P.head, kFP16, P.h, P.final_norm, nullptr);
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
#ifdef MSW_TRACE
    if (g_mk_trace) {
      unsigned long long g_;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_));
      g_mk_trace[8002] = g_;
      g_mk_trace[8003] = clock64();
    }
#endif
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
  const size_t attn = size_t(2) * 2 * 32 * P.D * 2 + size_t(G) * P.D * 4 + size_t(2) * P.D * 2 +
                      size_t(G) * 32 * 4;
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
  auto ok = [](int k) { return k % 128 == 0 && k <= 4 * 4 * kMkConsThreads * 2; };
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
