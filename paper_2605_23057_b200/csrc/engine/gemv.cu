// Decode GEMV (1..6 tokens) for the three weight formats, TMA-fed, on the
// tensor cores.
//
// HBM-bound: every weight byte is read once per step. Decode weights are
// stored "tile-fragment" (TF): 16-row tiles, each a contiguous run of 512-byte
// chunks, a chunk being one 16-byte mma.sync A fragment per lane:
//   FP16 : m16n8k16 f16 -> f32, chunk = 16 rows x 16 k
//   INT8 : m16n8k32 s8 -> s32 (exact), chunk = 16 rows x 32 k
//   W4   : m16n8k16 f16, chunk = 16 rows x 64 k (4 k16 steps). Dequant is ONE
//          lop3 per fp16 pair and no subtraction: even k16 steps feed (1024 + q)
//          against x, odd steps feed (1024 + 16 q) against x/16 (so one shift
//          serves four lop3s); the per-group offset 1032*Sx_even + 72*Sx_odd
//          (activation sums from the prologue) is removed in fp32 before the
//          group scale: sum_k (q-8) x = D_even + D_odd - C_group.
// The 8 MMA columns carry up to 8 tokens (verify / tiny batches) at no cost.
//
// Per CTA (persistent, one per SM, a contiguous tile range): a producer warp
// streams the CTA's weights through an smem ring with cp.async.bulk (<= 16 KB
// stages, mbarrier full/empty) and starts BEFORE griddepcontrol.wait, so the
// ring fills while the previous kernel finishes (PDL); 8 consumer warps each
// take a slice of every stage, run the MMAs, and reduce the 16 x 8 tile across
// warps in smem at tile boundaries. The activation prologue (RMSNorm, fp16
// rounding / per-token int8 quantisation) runs once per CTA into smem.
#include "kernels.cuh"
#include "mma_frag.cuh"

namespace msw {
#ifdef MSW_TRACE
__device__ unsigned long long* g_msw_trace = nullptr;
__device__ __forceinline__ unsigned long long* msw_trace_buf() { return g_msw_trace; }
#endif
namespace {

constexpr int kConsumers = 16;
constexpr int kThreads = (kConsumers + 2) * 32;  // + producer warp + epilogue warp
constexpr int kConsThreads = kConsumers * 32;
constexpr int kChunkBytes = 512;

// The head of the NEXT decode linear's weight stream, per CTA: once a CTA's
// producer has issued its last ring stage it prefetches into L2 the first
// w_bytes of the slice CTA blockIdx.x of the next GEMV will stream (and that
// CTA's scale block), so the next kernel's ring starts on L2 hits instead of
// a cold HBM round trip. The bytes are the ones the next kernel reads anyway:
// no extra HBM traffic, only earlier.
struct L2Next {
  const uint8_t* w = nullptr;
  const uint8_t* s = nullptr;
  uint32_t w_stride = 0, w_bytes = 0, w_total = 0;
  uint32_t s_stride = 0, s_bytes = 0, s_total = 0;
  int ncta = 0;
};

__device__ __forceinline__ void l2_next_prefetch(const L2Next& nx) {
  if (int(blockIdx.x) >= nx.ncta) return;
  const uint32_t wo = blockIdx.x * nx.w_stride;
  if (nx.w_bytes && wo < nx.w_total) prefetch_l2(nx.w + wo, min(nx.w_bytes, nx.w_total - wo));
  const uint32_t so = blockIdx.x * nx.s_stride;
  if (nx.s_bytes && so < nx.s_total) prefetch_l2(nx.s + so, min(nx.s_bytes, nx.s_total - so));
}
constexpr int kMaxStages = 8;
constexpr int kSmemBudget = 190 * 1024;

template <int FMT>
struct TF {
  static constexpr int kChunkK = FMT == kFP16 ? 16 : (FMT == kINT8 ? 32 : 64);
  static constexpr int kMinChunksPerWarp = FMT == kW4 ? 2 : 1;  // a W4 scale group is 2 chunks
};

// Consumer-only block reductions (named barrier 1 over the consumer warps).
__device__ __forceinline__ float cons_sum(float v, float* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  named_sync(1, kConsThreads);
  if (lane == 0) red[warp] = v;
  named_sync(1, kConsThreads);
  const float t = lane < kConsumers ? red[lane] : 0.0f;
  return warp_sum(t);
}
__device__ __forceinline__ float cons_max(float v, float* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_max(v);
  named_sync(1, kConsThreads);
  if (lane == 0) red[warp] = v;
  named_sync(1, kConsThreads);
  const float t = lane < kConsumers ? red[lane] : -3.402823466e38f;
  return warp_max(t);
}

// Register slots per thread of the register-resident prologues: float4 i =
// tid + 512 j, j < kW4ProRegs (k <= 16384).
constexpr int kW4ProRegs = 8;
// RMSNorm weights of the decode prologues (model constants): thread tid's
// float4 slots i = tid + 512 j, loaded into registers BEFORE griddepcontrol.wait
// so the only global load left after it is x (a gamma load after the norm
// reduction was a second dependent L2 round trip on every normed linear).
template <int PRO>
__device__ __forceinline__ void preload_gamma(const half* __restrict__ gamma, int k,
                                              uint2 (&gpre)[kW4ProRegs]) {
  if constexpr (PRO == kProNorm) {
    if (k > kW4ProRegs * 4 * kConsThreads) return;
#pragma unroll
    for (int j = 0; j < kW4ProRegs; ++j) {
      const int i = threadIdx.x + j * kConsThreads;
      if (i < k / 4) gpre[j] = reinterpret_cast<const uint2*>(gamma)[i];
    }
  }
}
__device__ __forceinline__ float4 apply_norm(float4 a, float r, uint2 gv) {
  const float2 g0 = __half22float2(*reinterpret_cast<const half2*>(&gv.x));
  const float2 g1 = __half22float2(*reinterpret_cast<const half2*>(&gv.y));
  a.x = (a.x * r) * g0.x;
  a.y = (a.y * r) * g0.y;
  a.z = (a.z * r) * g1.x;
  a.w = (a.w * r) * g1.y;
  return a;
}

// x fp32 [T, k] -> smem: fp16 [NT][k] (FP16 / W4) or int8 [NT][k] + scale.
// W4 per-group activation offsets (corr region after the two fp16 copies):
// GPTQ (zero point 8): C[t][g] = 1032 * Se + 72 * So, one float per group;
// AWQ (zp: zero point per row and group): B[t][g] = 1024 * Se + 64 * So and
// S[t][g] = Se + So, the row's offset being B + z * S (Se / So: sums of the
// fp16-rounded x over the even / odd k16 steps of the group).
template <int FMT, int PRO, int NT>
__device__ __forceinline__ void prologue(const float* __restrict__ x, const half* __restrict__ gamma,
                                         float eps, int k, int T, uint8_t* xs, float* red,
                                         float* xscale, bool zp = false) {
  const int tid = threadIdx.x;
  for (int t = 0; t < (FMT == kW4 ? NT : T); ++t) {  // FP16 / INT8 stage the T real rows only
    const int bytes = FMT == kINT8 ? k : 2 * k;
    if (t >= T) {  // padding token columns: never stored, but keep them finite
      for (int i = tid; i < bytes / 16; i += kConsThreads)
        reinterpret_cast<uint4*>(xs + size_t(t) * bytes)[i] = make_uint4(0, 0, 0, 0);
      if (tid == 0) xscale[t] = 0.0f;
      continue;
    }
    const float4* xt = reinterpret_cast<const float4*>(x + size_t(t) * k);
    const int k4 = k / 4;
    float r = 1.0f;
    if (PRO == kProNorm) {
      float ss = 0.0f;
      for (int i = tid; i < k4; i += kConsThreads) {
        const float4 v = xt[i];
        ss = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, ss))));
      }
      ss = cons_sum(ss, red);
      r = 1.0f / sqrtf(ss / float(k) + eps);
    }
    auto act4 = [&](int i) -> float4 {
      float4 v = xt[i];
      if (PRO == kProNorm) {
        const half2* gm = reinterpret_cast<const half2*>(gamma) + 2 * i;
        const float2 g0 = __half22float2(gm[0]), g1 = __half22float2(gm[1]);
        v.x = (v.x * r) * g0.x;
        v.y = (v.y * r) * g0.y;
        v.z = (v.z * r) * g1.x;
        v.w = (v.w * r) * g1.y;
      }
      return v;
    };
    if (FMT == kINT8) {
      float amax = 0.0f;
      for (int i = tid; i < k4; i += kConsThreads) {
        const float4 v = act4(i);
        amax = fmaxf(amax, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
      }
      amax = cons_max(amax, red);
      const float s = amax / 127.0f;
      int8_t* xq = reinterpret_cast<int8_t*>(xs + size_t(t) * k);
      auto q = [&](float v) -> int8_t {
        const float u = amax > 0.0f ? rintf(v / s) : 0.0f;
        return static_cast<int8_t>(fminf(fmaxf(u, -127.0f), 127.0f));
      };
      for (int i = tid; i < k4; i += kConsThreads) {
        const float4 v = act4(i);
        // 4 consecutive k stay together: one char4 at its permuted slot
        *reinterpret_cast<char4*>(xq + perm_i8(4 * i)) = make_char4(q(v.x), q(v.y), q(v.z), q(v.w));
      }
      if (tid == 0) xscale[t] = s;
    } else {
      half* xh = reinterpret_cast<half*>(xs + size_t(t) * 2 * k);
      half* xh16 = reinterpret_cast<half*>(xs + size_t(NT) * 2 * k + size_t(t) * 2 * k);
      for (int i = tid; i < k4; i += kConsThreads) {
        const float4 v = act4(i);
        const half2 lo = __floats2half2_rn(v.x, v.y), hi = __floats2half2_rn(v.z, v.w);
        // pairs (k, k+1) stay together at their permuted slot
        *reinterpret_cast<half2*>(xh + perm_f16(4 * i)) = lo;
        *reinterpret_cast<half2*>(xh + perm_f16(4 * i + 2)) = hi;
        if (FMT == kW4) {  // x/16 copy (exact power-of-two scaling) for the odd k16 steps
          *reinterpret_cast<half2*>(xh16 + perm_f16(4 * i)) = __hmul2(lo, __float2half2_rn(0.0625f));
          *reinterpret_cast<half2*>(xh16 + perm_f16(4 * i + 2)) = __hmul2(hi, __float2half2_rn(0.0625f));
        }
      }
      if (FMT == kW4) {
        named_sync(1, kConsThreads);
        // per-group offsets C = 1032 * sum(x | even k16 steps) + 72 * sum(x | odd k16 steps)
        const int groups = k / kW4Group;
        float* corr = reinterpret_cast<float*>(xs + size_t(NT) * 4 * k) + size_t(t) * groups;
        const int lane = tid & 31, warp = tid >> 5;
        for (int grp = warp; grp < groups; grp += kConsumers) {
          double se = 0.0, so = 0.0;
          for (int i = lane; i < kW4Group; i += 32) {
            const double v = __half2float(xh[perm_f16(grp * kW4Group + i)]);
            if ((i & 31) < 16) se += v;
            else so += v;
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            se += __shfl_xor_sync(0xffffffffu, se, o);
            so += __shfl_xor_sync(0xffffffffu, so, o);
          }
          if (lane == 0) {
            if (zp) {
              corr[grp] = float(1024.0 * se + 64.0 * so);
              corr[size_t(NT) * groups + grp] = float(se + so);
            } else {
              corr[grp] = float(1032.0 * se + 72.0 * so);
            }
          }
        }
      }
    }
    named_sync(1, kConsThreads);
  }
}

// Multi-token FP16 / INT8 prologue (verify, small continuous-batching
// steps): every token's statistics in ONE pass and one block reduction
// (instead of one pass and two barriers per token in sequence), then one
// conversion pass over all tokens. red2: [2][NT][kConsumers] floats.
template <int FMT, int PRO, int NT>
__device__ __forceinline__ void prologue_multi(const float* __restrict__ x,
                                               const half* __restrict__ gamma, float eps, int k,
                                               int T, uint8_t* xs, float* red2, float* xscale,
                                               const uint2 (&gpre)[kW4ProRegs]) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k4 = k / 4;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  float* redm = red2;                       // [NT][kConsumers]
  float* redx = red2 + NT * kConsumers;     // [NT][kConsumers]
  float r[NT];
#pragma unroll
  for (int t = 0; t < NT; ++t) r[t] = 1.0f;
  if (PRO == kProNorm) {
    float ss[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) ss[t] = 0.0f;
    for (int i = tid; i < k4; i += kConsThreads) {
#pragma unroll
      for (int t = 0; t < NT; ++t)
        if (t < T) {
          const float4 v = x4[size_t(t) * k4 + i];
          ss[t] = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, ss[t]))));
        }
    }
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const float w = warp_sum(ss[t]);
      if (lane == 0) redm[t * kConsumers + warp] = w;
    }
    named_sync(1, kConsThreads);
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const float v = warp_sum(lane < kConsumers ? redm[t * kConsumers + lane] : 0.0f);
      r[t] = 1.0f / sqrtf(v / float(k) + eps);
    }
  }
  auto act4 = [&](int t, int i) -> float4 {
    float4 v = x4[size_t(t) * k4 + i];
    if (PRO == kProNorm) {
      const half2* gm = reinterpret_cast<const half2*>(gamma) + 2 * i;
      const float2 g0 = __half22float2(gm[0]), g1 = __half22float2(gm[1]);
      v.x = (v.x * r[t]) * g0.x;
      v.y = (v.y * r[t]) * g0.y;
      v.z = (v.z * r[t]) * g1.x;
      v.w = (v.w * r[t]) * g1.y;
    }
    return v;
  };
  if (FMT == kINT8) {
    float am[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) am[t] = 0.0f;
    for (int i = tid; i < k4; i += kConsThreads) {
#pragma unroll
      for (int t = 0; t < NT; ++t)
        if (t < T) {
          const float4 v = act4(t, i);
          am[t] = fmaxf(am[t], fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
        }
    }
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const float w = warp_max(am[t]);
      if (lane == 0) redx[t * kConsumers + warp] = w;
    }
    named_sync(1, kConsThreads);
#pragma unroll
    for (int t = 0; t < NT; ++t)
      am[t] = warp_max(lane < kConsumers ? redx[t * kConsumers + lane] : 0.0f);
    for (int i = tid; i < k4; i += kConsThreads) {
#pragma unroll
      for (int t = 0; t < NT; ++t)
        if (t < T) {
          const float4 v = act4(t, i);
          const float sc = am[t] / 127.0f;
          auto q = [&](float u) -> int8_t {
            const float w = am[t] > 0.0f ? rintf(u / sc) : 0.0f;
            return static_cast<int8_t>(fminf(fmaxf(w, -127.0f), 127.0f));
          };
          *reinterpret_cast<char4*>(xs + size_t(t) * k + perm_i8(4 * i)) =
              make_char4(q(v.x), q(v.y), q(v.z), q(v.w));
        }
    }
    if (tid < NT) xscale[tid] = tid < T ? am[tid] / 127.0f : 0.0f;
  } else if (PRO == kProNorm && k4 <= kW4ProRegs * kConsThreads) {
    // FP16, normed: the RMSNorm weights come from registers (preload_gamma)
#pragma unroll
    for (int j = 0; j < kW4ProRegs; ++j) {
      const int i = tid + j * kConsThreads;
      if (i >= k4) break;
#pragma unroll
      for (int t = 0; t < NT; ++t)
        if (t < T) {
          const float4 v = apply_norm(x4[size_t(t) * k4 + i], r[t], gpre[j]);
          half* xh = reinterpret_cast<half*>(xs + size_t(t) * 2 * k);
          *reinterpret_cast<half2*>(xh + perm_f16(4 * i)) = __floats2half2_rn(v.x, v.y);
          *reinterpret_cast<half2*>(xh + perm_f16(4 * i + 2)) = __floats2half2_rn(v.z, v.w);
        }
    }
  } else {
    for (int i = tid; i < k4; i += kConsThreads) {
#pragma unroll
      for (int t = 0; t < NT; ++t)
        if (t < T) {
          const float4 v = act4(t, i);
          half* xh = reinterpret_cast<half*>(xs + size_t(t) * 2 * k);
          *reinterpret_cast<half2*>(xh + perm_f16(4 * i)) = __floats2half2_rn(v.x, v.y);
          *reinterpret_cast<half2*>(xh + perm_f16(4 * i + 2)) = __floats2half2_rn(v.z, v.w);
        }
    }
  }
  named_sync(1, kConsThreads);
}

// Batch-1 W4 prologue (k <= 16384): x stays in registers between the RMSNorm
// reduction and the conversion, and the per-group offsets are reduced inside
// the conversion loop. Thread tid converts float4 i = tid + 512 j, so warp w
// covers exactly k in [128 (w + 16 j), +128) = one scale group per j, and
// lane bit 2 is the k16-step parity: four xor-shuffles (1, 2, 8, 16) leave
// the even-step sum in lane 0 and the odd-step sum in lane 4.
// Group sums are fp32 (pairwise tree over the fp16-rounded x).
// Batch-1 FP16 prologue (k <= 16384): x read once into registers, gamma from
// preload_gamma; the same arithmetic as prologue<kFP16, PRO, 1>. (The INT8
// equivalent measured 0.25% slower per 8B decode token than the generic
// prologue, 1.788 vs 1.784 ms, and is not used.)
template <int PRO>
__device__ __forceinline__ void prologue_t1_f16(const float* __restrict__ x,
                                                const uint2 (&gpre)[kW4ProRegs], float eps, int k,
                                                uint8_t* xs, float* red) {
  const int tid = threadIdx.x;
  const int k4 = k / 4;
  const float4* xt = reinterpret_cast<const float4*>(x);
  float4 v[kW4ProRegs];
#pragma unroll
  for (int j = 0; j < kW4ProRegs; ++j)
    if (tid + j * kConsThreads < k4) v[j] = xt[tid + j * kConsThreads];
  if (PRO == kProNorm) {
    float ss = 0.0f;
#pragma unroll
    for (int j = 0; j < kW4ProRegs; ++j)
      if (tid + j * kConsThreads < k4)
        ss = fmaf(v[j].x, v[j].x, fmaf(v[j].y, v[j].y, fmaf(v[j].z, v[j].z, fmaf(v[j].w, v[j].w, ss))));
    ss = cons_sum(ss, red);
    const float r = 1.0f / sqrtf(ss / float(k) + eps);
#pragma unroll
    for (int j = 0; j < kW4ProRegs; ++j)
      if (tid + j * kConsThreads < k4) v[j] = apply_norm(v[j], r, gpre[j]);
  }
  half* xh = reinterpret_cast<half*>(xs);
#pragma unroll
  for (int j = 0; j < kW4ProRegs; ++j) {
    const int i = tid + j * kConsThreads;
    if (i < k4) {
      *reinterpret_cast<half2*>(xh + perm_f16(4 * i)) = __floats2half2_rn(v[j].x, v[j].y);
      *reinterpret_cast<half2*>(xh + perm_f16(4 * i + 2)) = __floats2half2_rn(v[j].z, v[j].w);
    }
  }
  named_sync(1, kConsThreads);
}

template <int PRO>
__device__ __forceinline__ void prologue_w4_t1(const float* __restrict__ x,
                                               const uint2 (&gpre)[kW4ProRegs], float eps, int k,
                                               uint8_t* xs, float* red, bool zp) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k4 = k / 4;
  const float4* xt = reinterpret_cast<const float4*>(x);
  float4 v[kW4ProRegs];
#pragma unroll
  for (int j = 0; j < kW4ProRegs; ++j)
    if (tid + j * kConsThreads < k4) v[j] = xt[tid + j * kConsThreads];
  float r = 1.0f;
  if (PRO == kProNorm) {
    float ss = 0.0f;
#pragma unroll
    for (int j = 0; j < kW4ProRegs; ++j)
      if (tid + j * kConsThreads < k4)
        ss = fmaf(v[j].x, v[j].x, fmaf(v[j].y, v[j].y, fmaf(v[j].z, v[j].z, fmaf(v[j].w, v[j].w, ss))));
    ss = cons_sum(ss, red);
    r = 1.0f / sqrtf(ss / float(k) + eps);
  }
  half* xh = reinterpret_cast<half*>(xs);
  half* xh16 = reinterpret_cast<half*>(xs + size_t(2) * k);
  float* corr = reinterpret_cast<float*>(xs + size_t(4) * k);
  const half2 sixteenth = __float2half2_rn(0.0625f);
#pragma unroll
  for (int j = 0; j < kW4ProRegs; ++j) {
    const int i = tid + j * kConsThreads;
    if (warp * 32 + j * kConsThreads >= k4) continue;  // warp-uniform: k4 % 32 == 0
    float4 a = v[j];
    if (PRO == kProNorm) a = apply_norm(a, r, gpre[j]);
    const half2 lo = __floats2half2_rn(a.x, a.y), hi = __floats2half2_rn(a.z, a.w);
    *reinterpret_cast<half2*>(xh + perm_f16(4 * i)) = lo;
    *reinterpret_cast<half2*>(xh + perm_f16(4 * i + 2)) = hi;
    *reinterpret_cast<half2*>(xh16 + perm_f16(4 * i)) = __hmul2(lo, sixteenth);
    *reinterpret_cast<half2*>(xh16 + perm_f16(4 * i + 2)) = __hmul2(hi, sixteenth);
    const float2 lf = __half22float2(lo), hf = __half22float2(hi);
    float gs = (lf.x + lf.y) + (hf.x + hf.y);
    gs += __shfl_xor_sync(0xffffffffu, gs, 1);
    gs += __shfl_xor_sync(0xffffffffu, gs, 2);
    gs += __shfl_xor_sync(0xffffffffu, gs, 8);
    gs += __shfl_xor_sync(0xffffffffu, gs, 16);
    const float odd = __shfl_sync(0xffffffffu, gs, 4);
    if (lane == 0) {
      if (zp) {  // AWQ: base and group sum (see prologue)
        corr[warp + j * kConsumers] = 1024.0f * gs + 64.0f * odd;
        corr[k / kW4Group + warp + j * kConsumers] = gs + odd;
      } else {
        corr[warp + j * kConsumers] = 1032.0f * gs + 72.0f * odd;
      }
    }
  }
  named_sync(1, kConsThreads);
}

template <int EPI>
__device__ __forceinline__ void store_pair(float* y, int n, int t, int row, float v0, float v1) {
  if (EPI == kEpiStore) {
    y[size_t(t) * n + row] = v0;
    y[size_t(t) * n + row + 1] = v1;
  } else if (EPI == kEpiResid) {
    y[size_t(t) * n + row] += v0;
    y[size_t(t) * n + row + 1] += v1;
  } else {
    y[size_t(t) * (n / 2) + row / 2] = silu(v0) * v1;  // rows (2i, 2i+1) = (gate_i, up_i)
  }
}

// Batch-1 residual epilogue: the residual rows of the CTA's first kResPre
// tiles are read into registers right after griddepcontrol.wait (the stream
// is fully ordered there), so the final y += v of a tile is a store, not a
// dependent L2 round trip at the end of the kernel. Lane (row pair rp = lane
// / 4, q = lane % 4 == 0) owns rows 2 rp, 2 rp + 1 of every tile.
constexpr int kResPre = 4;
template <int EPI, int NT>
__device__ __forceinline__ void resid_prefetch(const float* y, int tile_begin, int ntile_cta,
                                               float2 (&rpre)[kResPre]) {
  if constexpr (EPI == kEpiResid && NT == 1) {
    const int lane = threadIdx.x & 31;
    if ((lane & 3) != 0) return;
#pragma unroll
    for (int i = 0; i < kResPre; ++i)
      if (i < ntile_cta) rpre[i] = *reinterpret_cast<const float2*>(y + (tile_begin + i) * 16 + 2 * (lane >> 2));
  }
}
// store_pair for one token, using the prefetched residual of tile i when held
template <int EPI>
__device__ __forceinline__ void store_pair_t1(float* y, int n, int i, int row, float v0, float v1,
                                              const float2 (&rpre)[kResPre]) {
  if (EPI == kEpiResid && i < kResPre) {
    float2 r = rpre[0];
#pragma unroll
    for (int u = 1; u < kResPre; ++u)
      if (i == u) r = rpre[u];
    *reinterpret_cast<float2*>(y + row) = make_float2(r.x + v0, r.y + v1);
  } else {
    store_pair<EPI>(y, n, 0, row, v0, v1);
  }
}

// Warp roles (one CTA per SM, a contiguous range of 16-row tiles):
//   warps 0..kConsumers-1 : consumers. Every contiguous 16 KB ring stage holds
//                           S chunks of one tile; warp w takes CPW of them.
//                           At a tile end each warp red.shared-adds its 16 x 8
//                           partial into one of two tile accumulators and
//                           arrives on that buffer's mbarrier (no CTA barrier).
//   warp kConsumers       : producer (cp.async.bulk ring, ahead of the PDL wait)
//   warp kConsumers + 1   : epilogue: waits for a tile's accumulator, applies
//                           the scales / SwiGLU / residual store, zeroes the
//                           buffer and hands it back.
template <int FMT, int PRO, int EPI, int NT, int S>
__global__ void __launch_bounds__(kThreads, 1)
    gemv_tf_kernel(const uint8_t* __restrict__ wtf, const void* __restrict__ ws, int n, int k,
                   const float* __restrict__ x, int T, const half* __restrict__ gamma, float eps,
                   float* __restrict__ y, int n_stages, const L2Next nx,
                   const uint8_t* __restrict__ wz) {
  using Acc = typename std::conditional<FMT == kINT8, int, float>::type;
  constexpr int CK = TF<FMT>::kChunkK;
  constexpr int CPW = (S / kConsumers) > TF<FMT>::kMinChunksPerWarp ? (S / kConsumers)
                                                                     : TF<FMT>::kMinChunksPerWarp;
  constexpr int ACTIVE = S / CPW;
  constexpr int STAGE_BYTES = S * kChunkBytes;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full[kMaxStages], empty[kMaxStages], sbar;
  __shared__ uint64_t tile_full[2], tile_free[2];
  __shared__ float red[32];
  __shared__ float red2[2 * NT * kConsumers];  // multi-token prologue reductions
  __shared__ float xscale[NT];
  __shared__ __align__(16) uint32_t part[2][kConsumers][16][8];  // per-warp tile partials
  __shared__ __align__(16) uint8_t zero_b[64];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int chunks_tile = k / CK;
  const int ntiles = n / 16;
  const int per_cta = (ntiles + gridDim.x - 1) / gridDim.x;
  const int tile_begin = blockIdx.x * per_cta;
  const int tile_end = min(ntiles, tile_begin + per_cta);
  const int ntile_cta = max(0, tile_end - tile_begin);
  const int stages_tile = chunks_tile / S;
  const int total_stages = ntile_cta * stages_tile;
  const int groups_k = k / kW4Group;
  const int rows = ntile_cta * 16;
  // FP16 / INT8 stage only the T real token rows (a 5-token FP16 verify at
  // K = 14336 keeps a 3-stage ring instead of 2); W4 keeps NT rows
  const bool zp = FMT == kW4 && wz != nullptr;  // AWQ zero points (W4 only)
  const int xbytes = FMT == kINT8 ? T * k
                                  : (FMT == kW4 ? NT * 4 * k + 2 * NT * (k / kW4Group) * 4 : T * 2 * k);
  const int zbytes = zp ? rows * groups_k : 0;  // uint8 [rows][groups] after the scales
  const int sbytes = (FMT == kW4 ? rows * groups_k * 2 : (FMT == kINT8 ? rows * 4 : 0)) + zbytes;
  uint8_t* xs = smem;
  uint8_t* sc_smem = smem + ((xbytes + 127) & ~127);
  uint8_t* ring = sc_smem + ((sbytes + 127) & ~127);

  if (threadIdx.x < 64) zero_b[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < n_stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], ACTIVE);
    }
    mbar_init(&sbar, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tile_full[b], ACTIVE * 32);  // every consumer lane publishes its own partial
      mbar_init(&tile_free[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kConsumers) {
    // producer: weights only, so it runs ahead of griddepcontrol.wait
    if (lane == 0 && total_stages > 0) {
      if (sbytes > 0) {
        const uint8_t* ssrc = static_cast<const uint8_t*>(ws) +
                              size_t(tile_begin) * 16 * (FMT == kW4 ? groups_k * 2 : 4);
        mbar_expect_tx(&sbar, sbytes);
        bulk_g2s(sc_smem, ssrc, sbytes - zbytes, &sbar);
        if (zp) bulk_g2s(sc_smem + (sbytes - zbytes), wz + size_t(tile_begin) * 16 * groups_k, zbytes, &sbar);
      }
      const uint8_t* src = wtf + size_t(tile_begin) * chunks_tile * kChunkBytes;
      int s = 0;
      uint32_t phase = 0;
      for (int st = 0; st < total_stages; ++st) {
        mbar_wait(&empty[s], phase ^ 1);
        // the consumers read this slot with generic-proxy loads; order those
        // reads (acquired through the empty barrier) before the async-proxy
        // bulk copy that overwrites it
        fence_proxy_async();
        mbar_expect_tx(&full[s], STAGE_BYTES);
        bulk_g2s(ring + size_t(s) * STAGE_BYTES, src + size_t(st) * STAGE_BYTES, STAGE_BYTES, &full[s]);
        if (++s == n_stages) {
          s = 0;
          phase ^= 1;
        }
      }
      l2_next_prefetch(nx);
    }
    pdl_wait();
    pdl_trigger();
    return;
  }
  if (warp == kConsumers + 1) {
    // epilogue warp: tile accumulators -> y (scales, SwiGLU pairing, residual)
    pdl_wait();
    pdl_trigger();
    float2 rpre[kResPre];
    resid_prefetch<EPI, NT>(y, tile_begin, ntile_cta, rpre);
    if (sbytes > 0 && total_stages > 0) mbar_wait(&sbar, 0);
    named_sync(3, kConsThreads + 32);  // prologue (xscale) is complete
    const float* sc_f = reinterpret_cast<const float*>(sc_smem);
    for (int i = 0; i < ntile_cta; ++i) {
      const int b = i & 1;
      mbar_wait(&tile_full[b], (i >> 1) & 1);
      const int tile = tile_begin + i;
      // 128 (row, col) values; lane handles rows 2*(lane>>3)+{0,1} (a pair), col lane & 7,
      // for row pairs lane>>3 in {0..3} and +4 in a second pass
      if (NT == 1) {
        // one token: compact [warp][16] column-0 partials; lane (row pair rp,
        // quarter q) sums a quarter of the active warps, then a fixed 4-lane
        // shuffle tree (integer sums stay exact)
        const uint32_t* p1 = &part[b][0][0][0];
        const int rp = lane >> 2, q = lane & 3;
        const int row = 2 * rp;
        Acc a0 = 0, a1 = 0;
        for (int w2 = q; w2 < ACTIVE; w2 += 4) {
          if (FMT == kINT8) {
            a0 += Acc(int(p1[w2 * 16 + row]));
            a1 += Acc(int(p1[w2 * 16 + row + 1]));
          } else {
            a0 += Acc(__uint_as_float(p1[w2 * 16 + row]));
            a1 += Acc(__uint_as_float(p1[w2 * 16 + row + 1]));
          }
        }
        a0 += __shfl_xor_sync(0xffffffffu, a0, 1);
        a1 += __shfl_xor_sync(0xffffffffu, a1, 1);
        a0 += __shfl_xor_sync(0xffffffffu, a0, 2);
        a1 += __shfl_xor_sync(0xffffffffu, a1, 2);
        if (q == 0) {
          if (FMT == kINT8 && EPI == kEpiRaw) {
            reinterpret_cast<int*>(y)[tile * 16 + row] = int(a0);
            reinterpret_cast<int*>(y)[tile * 16 + row + 1] = int(a1);
          } else {
            float v0 = float(a0), v1 = float(a1);
            if (FMT == kINT8) {
              const int lrr = i * 16 + row;
              v0 = (v0 * xscale[0]) * sc_f[lrr];
              v1 = (v1 * xscale[0]) * sc_f[lrr + 1];
            }
            store_pair_t1<EPI>(y, n, i, tile * 16 + row, v0, v1, rpre);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&tile_free[b]);
        continue;
      }
#pragma unroll
      for (int pass = 0; pass < (NT == 1 ? 0 : 2); ++pass) {
        const int rp = (lane >> 3) + pass * 4;  // row pair 0..7
        const int col = lane & 7;
        const int row = 2 * rp;
        float v0, v1;
        if (FMT == kINT8) {  // exact int32 across warps
          int i0 = 0, i1 = 0;
#pragma unroll 4
          for (int w2 = 0; w2 < ACTIVE; ++w2) {
            i0 += int(part[b][w2][row][col]);
            i1 += int(part[b][w2][row + 1][col]);
          }
          if (EPI == kEpiRaw) {  // test entry: the int32 accumulators themselves
            if (col < T) {
              reinterpret_cast<int*>(y)[size_t(col) * n + tile * 16 + row] = i0;
              reinterpret_cast<int*>(y)[size_t(col) * n + tile * 16 + row + 1] = i1;
            }
            continue;
          }
          v0 = float(i0);
          v1 = float(i1);
        } else {
          v0 = 0.f;
          v1 = 0.f;
#pragma unroll 4
          for (int w2 = 0; w2 < ACTIVE; ++w2) {
            v0 += __uint_as_float(part[b][w2][row][col]);
            v1 += __uint_as_float(part[b][w2][row + 1][col]);
          }
        }
        if (col < T) {
          if (FMT == kINT8) {
            const int lrr = i * 16 + row;
            v0 = (v0 * xscale[col]) * sc_f[lrr];
            v1 = (v1 * xscale[col]) * sc_f[lrr + 1];
          }
          store_pair<EPI>(y, n, col, tile * 16 + row, v0, v1);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&tile_free[b]);
    }
    return;
  }

  // consumers
  uint2 gpre[kW4ProRegs];
  constexpr bool kT1 = NT == 1 && FMT == kFP16;
  if (FMT == kFP16) preload_gamma<PRO>(gamma, k, gpre);
  pdl_wait();
  pdl_trigger();
  if constexpr (NT > 1 && FMT != kW4)
    prologue_multi<FMT, PRO, NT>(x, gamma, eps, k, T, xs, red2, xscale, gpre);
  else if (kT1 && k <= kW4ProRegs * 4 * kConsThreads)
    prologue_t1_f16<PRO>(x, gpre, eps, k, xs, red);
  else
    prologue<FMT, PRO, NT>(x, gamma, eps, k, T, xs, red, xscale, zp);
  named_sync(3, kConsThreads + 32);  // release the epilogue warp (xscale ready)
  const int g = lane >> 2, tq = lane & 3;
  const bool has_tok = g < T;  // this lane's MMA column is a real token
  if (sbytes > 0 && total_stages > 0) mbar_wait(&sbar, 0);
  const half* sc_h = reinterpret_cast<const half*>(sc_smem);   // W4 [rows][groups_k]
  const float* corr = reinterpret_cast<const float*>(xs + size_t(NT) * 4 * k);
  // B-fragment rows. MMA column g only feeds output column g, and columns >= T
  // are never stored, so lanes without a token read token 0's row (finite)
  // instead of a zero slot: loop-invariant bases, no per-load masking.
  const int brow = has_tok ? g : 0;
  const uint8_t* xrow = xs + size_t(brow) * (FMT == kINT8 ? k : 2 * k) + tq * 8;
  const uint8_t* xrow16 = xs + size_t(NT) * 2 * k + size_t(brow) * 2 * k + tq * 8;

  Acc acc[4] = {0, 0, 0, 0};
  Acc acc2[4] = {0, 0, 0, 0};
  float cg[2][4] = {};
  int s = 0;
  uint32_t phase = 0;
  int c_tile0 = 0, ti = 0;  // chunk offset within the tile, tile index within the CTA
  const int my_c0 = warp * CPW;
  for (int st = 0; st < total_stages; ++st) {
    mbar_wait(&full[s], phase);
    if (warp < ACTIVE) {
      const uint4* stage = reinterpret_cast<const uint4*>(ring + size_t(s) * STAGE_BYTES) +
                           my_c0 * 32 + lane;
      const int cbase = c_tile0 + my_c0;
      const int lr = ti * 16 + g;
#pragma unroll
      for (int j = 0; j < CPW; ++j) {
        const uint4 a4 = stage[j * 32];
        const int c = cbase + j;
        if (FMT == kFP16) {
          const uint2 b = *reinterpret_cast<const uint2*>(xrow + c * 32);
          const uint32_t a[4] = {a4.x, a4.y, a4.z, a4.w};
          if (j & 1) mma_f16(reinterpret_cast<float(&)[4]>(acc2), a, b.x, b.y);
          else mma_f16(reinterpret_cast<float(&)[4]>(acc), a, b.x, b.y);
        } else if (FMT == kINT8) {
          const uint2 b = *reinterpret_cast<const uint2*>(xrow + c * 32);
          const uint32_t a[4] = {a4.x, a4.y, a4.z, a4.w};
          if (j & 1) mma_s8(reinterpret_cast<int(&)[4]>(acc2), a, b.x, b.y);
          else mma_s8(reinterpret_cast<int(&)[4]>(acc), a, b.x, b.y);
        } else {
          const uint32_t wv[4] = {a4.x, a4.y, a4.z, a4.w};
          float (&cgr)[4] = cg[(j >> 1) & 1];  // group accumulator (compile-time index: j is unrolled)
#pragma unroll
          for (int p = 0; p < 2; ++p) {  // step 2p: (1024+q) vs x; step 2p+1: (1024+16q) vs x/16
            const uint32_t w0 = wv[2 * p], w1 = wv[2 * p + 1];
            const uint32_t w0s = w0 >> 8, w1s = w1 >> 8;
            const uint32_t a_lo[4] = {lop3_and_or(w0, 0x000F000Fu, 0x64006400u),
                                      lop3_and_or(w0s, 0x000F000Fu, 0x64006400u),
                                      lop3_and_or(w1, 0x000F000Fu, 0x64006400u),
                                      lop3_and_or(w1s, 0x000F000Fu, 0x64006400u)};
            const uint32_t a_hi[4] = {lop3_and_or(w0, 0x00F000F0u, 0x64006400u),
                                      lop3_and_or(w0s, 0x00F000F0u, 0x64006400u),
                                      lop3_and_or(w1, 0x00F000F0u, 0x64006400u),
                                      lop3_and_or(w1s, 0x00F000F0u, 0x64006400u)};
            const int kb = (c * 64 + p * 32) * 2;  // byte offset of the even step's 16-k block
            const uint2 be = *reinterpret_cast<const uint2*>(xrow + kb);
            const uint2 bo = *reinterpret_cast<const uint2*>(xrow16 + kb + 32);
            mma_f16(cgr, a_lo, be.x, be.y);
            mma_f16(cgr, a_hi, bo.x, bo.y);
          }
          if (j & 1) {  // end of a 128-k group (my_c0 and CPW are even)
            const int grp = c >> 1;
            const float slo = __half2float(sc_h[lr * groups_k + grp]);
            const float shi = __half2float(sc_h[(lr + 8) * groups_k + grp]);
            const int t0c = 2 * tq < NT ? 2 * tq : 0, t1c = 2 * tq + 1 < NT ? 2 * tq + 1 : 0;
            const float c0 = corr[t0c * groups_k + grp];
            const float c1 = corr[t1c * groups_k + grp];
            if (zp) {  // AWQ: row offsets B + z * S (zero point per row and group)
              const uint8_t* zs = sc_smem + rows * groups_k * 2;
              const float zlo = zs[lr * groups_k + grp], zhi = zs[(lr + 8) * groups_k + grp];
              const float s0 = corr[(NT + t0c) * groups_k + grp], s1 = corr[(NT + t1c) * groups_k + grp];
              acc[0] = fmaf(slo, cgr[0] - fmaf(zlo, s0, c0), acc[0]);
              acc[1] = fmaf(slo, cgr[1] - fmaf(zlo, s1, c1), acc[1]);
              acc[2] = fmaf(shi, cgr[2] - fmaf(zhi, s0, c0), acc[2]);
              acc[3] = fmaf(shi, cgr[3] - fmaf(zhi, s1, c1), acc[3]);
            } else {
              acc[0] = fmaf(slo, cgr[0] - c0, acc[0]);
              acc[1] = fmaf(slo, cgr[1] - c1, acc[1]);
              acc[2] = fmaf(shi, cgr[2] - c0, acc[2]);
              acc[3] = fmaf(shi, cgr[3] - c1, acc[3]);
            }
            cgr[0] = cgr[1] = cgr[2] = cgr[3] = 0.f;
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (++s == n_stages) {
      s = 0;
      phase ^= 1;
    }
    c_tile0 += S;
    if (c_tile0 == chunks_tile) {
      // tile complete: add this warp's partial into the tile accumulator (async)
      c_tile0 = 0;
      if (warp < ACTIVE) {
        const int b = ti & 1;
        if (ti >= 2) mbar_wait(&tile_free[b], ((ti >> 1) - 1) & 1);  // epilogue drained it
        uint32_t r4[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const Acc tot = acc[i] + acc2[i];
          r4[i] = FMT == kINT8 ? uint32_t(int(tot)) : __float_as_uint(float(tot));
        }
        if (NT == 1) {  // column 0 only: lanes tq == 0 hold rows g and g + 8
          uint32_t* p1 = &part[b][0][0][0] + warp * 16;
          if (tq == 0) {
            p1[g] = r4[0];
            p1[g + 8] = r4[2];
          }
        } else {
          uint32_t* pw = &part[b][warp][0][0];
          pw[g * 8 + 2 * tq] = r4[0];
          pw[g * 8 + 2 * tq + 1] = r4[1];
          pw[(g + 8) * 8 + 2 * tq] = r4[2];
          pw[(g + 8) * 8 + 2 * tq + 1] = r4[3];
        }
        // each lane's arrive releases its OWN partial stores
        mbar_arrive(&tile_full[b]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i] = acc2[i] = 0;
      ++ti;
    }
  }
}

// W4 decode GEMV, issue-lean variant (8B shapes: K = 4096 and K = 14336).
// The generic kernel above spends ~68 warp instructions per 1024 weights at
// 2 chunks per warp per stage (barrier / loop / tile bookkeeping dominate)
// and is issue-bound below the HBM rate even with L2-resident weights. Here:
//   * every warp takes CPW = 4 chunks (two 128-k groups) per stage, so the
//     per-stage overhead is amortised over 4096 weights;
//   * GW warp groups take alternate stages (GW = 2 for K = 14336: 16 KB
//     stages, 8 warps each), so all 16 warps stay busy when a 32 KB stage
//     does not divide the tile;
//   * when the tile is exactly one stage (K = 4096, XREG) each warp's k-slice
//     never changes: its B fragments (fp16 x and x/16) and its two group
//     offsets live in registers for the whole kernel, leaving one LDS.128 of
//     weights plus two scale loads per 4096 weights;
//   * a warp flushes its 16 x 8 tile partial when its slice moves to the next
//     tile (stages may straddle tiles in the GW = 2 configuration).
// Numerics as gemv_tf_kernel<kW4> (identical MMA operands, per-group fp32
// accumulation, correction subtracted before the group scale) except that a
// group's 8 MMAs run as two chains of 4 (low / high nibbles) summed at the
// group end: a different fp32 summation order, within the W4 bar.
template <int PRO, int EPI, int NT, int S, int GW, bool XREG, bool ZP>
__global__ void __launch_bounds__(kThreads, 1)
    gemv_w4_kernel(const uint8_t* __restrict__ wtf, const void* __restrict__ ws, int n, int k,
                   const float* __restrict__ x, int T, const half* __restrict__ gamma, float eps,
                   float* __restrict__ y, int n_stages, const L2Next nx,
                   const uint8_t* __restrict__ wz) {
  constexpr int WPG = kConsumers / GW;  // warps sharing one stage
  constexpr int CPW = S / WPG;          // chunks per warp per stage
  static_assert(CPW == 4, "two 128-k groups per warp per stage");
  constexpr int STAGE_BYTES = S * kChunkBytes;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full[kMaxStages], empty[kMaxStages], sbar;
  __shared__ uint64_t tile_full[2], tile_free[2];
  __shared__ float red[32];
  __shared__ float xscale[NT];
  __shared__ __align__(16) float part[2][kConsumers][16][8];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int chunks_tile = k / 64;
  const int ntiles = n / 16;
  const int per_cta = (ntiles + gridDim.x - 1) / gridDim.x;
  const int tile_begin = blockIdx.x * per_cta;
  const int tile_end = min(ntiles, tile_begin + per_cta);
  const int ntile_cta = max(0, tile_end - tile_begin);
  const int total_stages = ntile_cta * chunks_tile / S;
  const int groups_k = k / kW4Group;
  const int rows = ntile_cta * 16;
  // ZP (AWQ): zero points [rows][groups] after the scales, and the group sums S
  // after the offsets in the activation region. A template constant: the
  // GPTQ instantiation carries no zero-point work in its issue-bound loop.
  constexpr bool zp = ZP;
  const int xbytes = NT * 4 * k + (ZP ? 2 : 1) * NT * groups_k * 4;
  const int zbytes = zp ? rows * groups_k : 0;
  const int sbytes = rows * groups_k * 2 + zbytes;
  uint8_t* xs = smem;
  uint8_t* sc_smem = smem + ((xbytes + 127) & ~127);
  uint8_t* ring = sc_smem + ((sbytes + 127) & ~127);

  if (threadIdx.x == 0) {
    for (int s = 0; s < n_stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], WPG);
    }
    mbar_init(&sbar, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tile_full[b], kConsumers * 32);  // every consumer lane arrives
      mbar_init(&tile_free[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kConsumers) {  // producer: weights + scales only, ahead of the PDL wait
    if (lane == 0) MSW_TP(0);
    if (lane == 0 && total_stages > 0) {
      mbar_expect_tx(&sbar, sbytes);
      bulk_g2s(sc_smem, static_cast<const uint8_t*>(ws) + size_t(tile_begin) * 16 * groups_k * 2,
               sbytes - zbytes, &sbar);
      if (zp) bulk_g2s(sc_smem + (sbytes - zbytes), wz + size_t(tile_begin) * 16 * groups_k, zbytes, &sbar);
      const uint8_t* src = wtf + size_t(tile_begin) * chunks_tile * kChunkBytes;
      int s = 0;
      uint32_t phase = 0;
      for (int st = 0; st < total_stages; ++st) {
        mbar_wait(&empty[s], phase ^ 1);
        // the consumers read this slot with generic-proxy loads; order those
        // reads (acquired through the empty barrier) before the async-proxy
        // bulk copy that overwrites it
        fence_proxy_async();
        mbar_expect_tx(&full[s], STAGE_BYTES);
        bulk_g2s(ring + size_t(s) * STAGE_BYTES, src + size_t(st) * STAGE_BYTES, STAGE_BYTES,
                 &full[s]);
        if (st == n_stages - 1) MSW_TP(1);  // ring primed
        if (++s == n_stages) {
          s = 0;
          phase ^= 1;
        }
      }
      MSW_TP(2);  // last stage issued
      l2_next_prefetch(nx);
    }
    pdl_wait();
    pdl_trigger();
    return;
  }
  if (warp == kConsumers + 1) {  // epilogue: 16 per-warp partials -> y
    pdl_wait();
    pdl_trigger();
    float2 rpre[kResPre];
    resid_prefetch<EPI, NT>(y, tile_begin, ntile_cta, rpre);
    named_sync(3, kConsThreads + 32);
    for (int i = 0; i < ntile_cta; ++i) {
      const int b = i & 1;
      mbar_wait(&tile_full[b], (i >> 1) & 1);
      const int tile = tile_begin + i;
      if (NT == 1) {
        // one token: only column 0 exists (compact [warp][16] partials). Lane
        // (row pair rp, quarter q) sums warps 4q..4q+3 of rows 2rp, 2rp+1, and
        // a 4-lane shuffle tree finishes the 16-warp sum (fixed order)
        const float* p1 = &part[b][0][0][0];
        const int rp = lane >> 2, q = lane & 3;
        float v0 = 0.f, v1 = 0.f;
#pragma unroll
        for (int i2 = 0; i2 < kConsumers / 4; ++i2) {
          v0 += p1[(q * (kConsumers / 4) + i2) * 16 + 2 * rp];
          v1 += p1[(q * (kConsumers / 4) + i2) * 16 + 2 * rp + 1];
        }
        v0 += __shfl_xor_sync(0xffffffffu, v0, 1);
        v1 += __shfl_xor_sync(0xffffffffu, v1, 1);
        v0 += __shfl_xor_sync(0xffffffffu, v0, 2);
        v1 += __shfl_xor_sync(0xffffffffu, v1, 2);
        if (q == 0) store_pair_t1<EPI>(y, n, i, tile * 16 + 2 * rp, v0, v1, rpre);
      } else {
#pragma unroll
        for (int pass = 0; pass < 2; ++pass) {
          const int row = 2 * ((lane >> 3) + pass * 4);
          const int col = lane & 7;
          float v0 = 0.f, v1 = 0.f;
#pragma unroll
          for (int w2 = 0; w2 < kConsumers; ++w2) {
            v0 += part[b][w2][row][col];
            v1 += part[b][w2][row + 1][col];
          }
          if (col < T) store_pair<EPI>(y, n, col, tile * 16 + row, v0, v1);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&tile_free[b]);
      if (lane == 0 && i == 0) MSW_TP(8);  // first tile stored
    }
    if (lane == 0) MSW_TP(9);  // all tiles stored
    return;
  }

  // consumers
  uint2 gpre[kW4ProRegs];
  if (NT == 1) preload_gamma<PRO>(gamma, k, gpre);
  pdl_wait();
  if (threadIdx.x == 0) MSW_TP(3);  // dependency resolved
  pdl_trigger();
  if (NT == 1 && k <= kW4ProRegs * 4 * kConsThreads)
    prologue_w4_t1<PRO>(x, gpre, eps, k, xs, red, zp);
  else
    prologue<kW4, PRO, NT>(x, gamma, eps, k, T, xs, red, xscale, zp);
  if (threadIdx.x == 0) MSW_TP(4);  // activations staged
  named_sync(3, kConsThreads + 32);
  const int g = lane >> 2, tq = lane & 3;
  const int gw = warp / WPG, wi = warp % WPG;
  const int brow = g < T ? g : 0;
  const uint8_t* xrow = xs + size_t(brow) * 2 * k + tq * 8;
  const uint8_t* xrow16 = xs + size_t(NT) * 2 * k + size_t(brow) * 2 * k + tq * 8;
  const half* sc_h = reinterpret_cast<const half*>(sc_smem);
  const float* corr = reinterpret_cast<const float*>(xs + size_t(NT) * 4 * k);
  const int tc0 = 2 * tq < NT ? 2 * tq : 0, tc1 = 2 * tq + 1 < NT ? 2 * tq + 1 : 0;
  // XREG: this warp's k-slice is chunks [wi*CPW, wi*CPW + CPW) of every tile
  uint2 bx[XREG ? CPW : 1][2][2];
  float cx[XREG ? CPW / 2 : 1][2];
  float sx[XREG ? CPW / 2 : 1][2];  // zp: the groups' activation sums S
  if (XREG) {
#pragma unroll
    for (int j = 0; j < CPW; ++j)
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const int kb = ((wi * CPW + j) * 64 + p * 32) * 2;
        bx[XREG ? j : 0][p][0] = *reinterpret_cast<const uint2*>(xrow + kb);
        bx[XREG ? j : 0][p][1] = *reinterpret_cast<const uint2*>(xrow16 + kb + 32);
      }
#pragma unroll
    for (int jj = 0; jj < CPW / 2; ++jj) {
      const int grp = (wi * CPW) / 2 + jj;
      cx[XREG ? jj : 0][0] = corr[tc0 * groups_k + grp];
      cx[XREG ? jj : 0][1] = corr[tc1 * groups_k + grp];
      sx[XREG ? jj : 0][0] = zp ? corr[(NT + tc0) * groups_k + grp] : 0.f;
      sx[XREG ? jj : 0][1] = zp ? corr[(NT + tc1) * groups_k + grp] : 0.f;
    }
  }
  if (total_stages > 0) mbar_wait(&sbar, 0);

  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  int cur = -1;  // tile (CTA-local) the accumulator belongs to
  // ring position of this warp's first stage; advanced incrementally by GW
  int slot = gw % n_stages;
  uint32_t phase = (gw / n_stages) & 1;
  auto flush = [&](int ti) {
    const int b = ti & 1;
    if (ti >= 2) mbar_wait(&tile_free[b], ((ti >> 1) - 1) & 1);
    if (NT == 1) {  // column 0 only: lanes tq == 0 hold rows g and g + 8
      float* p1 = &part[b][0][0][0] + warp * 16;
      if (tq == 0) {
        p1[g] = acc[0];
        p1[g + 8] = acc[2];
      }
    } else {
      float* pw = &part[b][warp][0][0];
      *reinterpret_cast<float2*>(pw + g * 8 + 2 * tq) = make_float2(acc[0], acc[1]);
      *reinterpret_cast<float2*>(pw + (g + 8) * 8 + 2 * tq) = make_float2(acc[2], acc[3]);
    }
    mbar_arrive(&tile_full[b]);  // per-lane release of its own stores (see gemv_tf_kernel)
    acc[0] = acc[1] = acc[2] = acc[3] = 0.f;
  };
#pragma unroll 1
  for (int st = gw; st < total_stages; st += GW) {
    const int gc = st * S + wi * CPW;  // chunk index in this CTA's stream
    const int ti = XREG ? st : gc / chunks_tile;  // XREG: one tile per stage
    const int c0 = XREG ? wi * CPW : gc - ti * chunks_tile;
    if (ti != cur) {
      if (cur >= 0) flush(cur);
      cur = ti;
    }
    mbar_wait(&full[slot], phase);
    if (threadIdx.x == 0 && st == 0) MSW_TP(5);  // first stage consumed
    if (threadIdx.x == 0 && st == n_stages) MSW_TP(6);  // ring wrapped once
    const uint4* stage = reinterpret_cast<const uint4*>(ring + size_t(slot) * STAGE_BYTES) +
                         wi * CPW * 32 + lane;
    uint4 a4[CPW];
#pragma unroll
    for (int j = 0; j < CPW; ++j) a4[j] = stage[j * 32];
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);  // operands are in registers
    slot += GW;
    if (slot >= n_stages) {
      slot -= n_stages;
      phase ^= 1;
    }
    const int lr = ti * 16 + g;
#pragma unroll
    for (int jj = 0; jj < CPW / 2; ++jj) {
      // two accumulator chains per group (low / high nibbles): the group's
      // 8 dependent MMAs become 2 x 4, halving the MMA latency chain
      float cg[4] = {0.f, 0.f, 0.f, 0.f}, ch[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int j = 2 * jj; j < 2 * jj + 2; ++j) {
        const uint32_t wv[4] = {a4[j].x, a4[j].y, a4[j].z, a4[j].w};
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          const uint32_t w0 = wv[2 * p], w1 = wv[2 * p + 1];
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
            const int kb = ((c0 + j) * 64 + p * 32) * 2;
            be = *reinterpret_cast<const uint2*>(xrow + kb);
            bo = *reinterpret_cast<const uint2*>(xrow16 + kb + 32);
          }
          mma_f16(cg, a_lo, be.x, be.y);
          mma_f16(ch, a_hi, bo.x, bo.y);
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) cg[i] += ch[i];
      const int grp = (c0 >> 1) + jj;
      const float slo = __half2float(sc_h[lr * groups_k + grp]);
      const float shi = __half2float(sc_h[(lr + 8) * groups_k + grp]);
      float k0, k1;
      if (XREG) {
        k0 = cx[XREG ? jj : 0][0];
        k1 = cx[XREG ? jj : 0][1];
      } else {
        k0 = corr[tc0 * groups_k + grp];
        k1 = corr[tc1 * groups_k + grp];
      }
      if (zp) {  // AWQ: the row's offset is B + z * S (zero point per row and group)
        const uint8_t* zs = sc_smem + rows * groups_k * 2;
        const float zlo = zs[lr * groups_k + grp], zhi = zs[(lr + 8) * groups_k + grp];
        const float s0 = XREG ? sx[XREG ? jj : 0][0] : corr[(NT + tc0) * groups_k + grp];
        const float s1 = XREG ? sx[XREG ? jj : 0][1] : corr[(NT + tc1) * groups_k + grp];
        acc[0] = fmaf(slo, cg[0] - fmaf(zlo, s0, k0), acc[0]);
        acc[1] = fmaf(slo, cg[1] - fmaf(zlo, s1, k1), acc[1]);
        acc[2] = fmaf(shi, cg[2] - fmaf(zhi, s0, k0), acc[2]);
        acc[3] = fmaf(shi, cg[3] - fmaf(zhi, s1, k1), acc[3]);
      } else {
        acc[0] = fmaf(slo, cg[0] - k0, acc[0]);
        acc[1] = fmaf(slo, cg[1] - k1, acc[1]);
        acc[2] = fmaf(shi, cg[2] - k0, acc[2]);
        acc[3] = fmaf(shi, cg[3] - k1, acc[3]);
      }
    }
  }
  if (cur >= 0) flush(cur);
  if (threadIdx.x == 0) MSW_TP(7);  // warp 0 done
}

// --------------------------------------------------------------- repacking
// Row-major source -> tile-fragment layout. Source formats:
//   FP16: half [n][k]; INT8: int8 [n][k]; W4: row-packed words [n][k/8]
//   (nibble position (i>>1) + 4*(i&1) for element i of a word).
__global__ void repack_tf_kernel(int fmt, const uint8_t* __restrict__ src, int n, int k,
                                 uint8_t* __restrict__ dst) {
  const int ck = fmt == kFP16 ? 16 : (fmt == kINT8 ? 32 : 64);
  const int chunks_tile = k / ck;
  const long long words = (long long)(n / 16) * chunks_tile * 32 * 4;  // 32-bit words
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < words;
       i += (long long)gridDim.x * blockDim.x) {
    const int reg = int(i & 3);  // A fragment register a0..a3 (W4: k16 step)
    const int lane = int((i >> 2) & 31);
    const long long tc = i >> 7;
    const int c = int(tc % chunks_tile);
    const int tile = int(tc / chunks_tile);
    const int g = lane >> 2, tq = lane & 3;
    uint32_t word = 0;
    if (fmt == kFP16) {
      const int row = tile * 16 + g + ((reg & 1) ? 8 : 0);
      const int kk = c * 16 + 2 * tq + ((reg & 2) ? 8 : 0);
      word = *reinterpret_cast<const uint32_t*>(src + (size_t(row) * k + kk) * 2);
    } else if (fmt == kINT8) {
      const int row = tile * 16 + g + ((reg & 1) ? 8 : 0);
      const int kk = c * 32 + 4 * tq + ((reg & 2) ? 16 : 0);
      word = *reinterpret_cast<const uint32_t*>(src + size_t(row) * k + kk);
    } else {
      // word `reg` = 2p + h of the chunk (p: step pair (2p, 2p+1); h: 0 -> fragment
      // regs a0/a1 (k base 2tq), 1 -> a2/a3 (k base 2tq + 8)). Nibble position ->
      // (step, fragment reg, lo/hi):
      //   pos0/pos4: step 2p,   row g,   k, k+1      pos2/pos6: step 2p,   row g+8, k, k+1
      //   pos1/pos5: step 2p+1, row g,   k, k+1      pos3/pos7: step 2p+1, row g+8, k, k+1
      const uint32_t* sw = reinterpret_cast<const uint32_t*>(src);
      const int p = reg >> 1, h = reg & 1;
#pragma unroll
      for (int pos = 0; pos < 8; ++pos) {
        const int step = 2 * p + (pos & 1);
        const int row = tile * 16 + g + ((pos & 2) ? 8 : 0);
        const int kk = c * 64 + step * 16 + 2 * tq + (h ? 8 : 0) + (pos >> 2);
        const uint32_t w = sw[size_t(row) * (k / 8) + kk / 8];
        const int si = kk & 7;
        const uint32_t q = (w >> (4 * ((si >> 1) + 4 * (si & 1)))) & 0xF;
        word |= q << (4 * pos);
      }
    }
    reinterpret_cast<uint32_t*>(dst)[i] = word;
  }
}

// L2 prefetch descriptor of the linear launched after the current one; set by
// launch_gemv for the duration of one launch (host-thread local, the launch
// captures it by value, so graph capture records it too).
thread_local L2Next t_next;

// Enabled behind W4 GEMVs only (128 KB per CTA: W4 decode 1.620 -> 1.588
// ms/token). FP16 and INT8 already run near the HBM rate, where the early
// bytes compete with the current stream: FP16 2.668 -> 2.72 ms, INT8 flat at
// 32 KB and worse above (scripts/l2next_ab.sh). MSW_L2NEXT_KB overrides.
L2Next make_l2_next(int cur_fmt, const LinearW* nw) {
  L2Next nx;
  static const long env_kb = [] {
    const char* v = diag_env("MSW_L2NEXT_KB");
    return v ? std::atol(v) : -1L;
  }();
  const long kb = env_kb >= 0 ? env_kb : (cur_fmt == kW4 ? 128L : 0L);
  if (!nw || !nw->w_tf || kb <= 0) return nx;
  const int ck = nw->fmt == kFP16 ? 16 : (nw->fmt == kINT8 ? 32 : 64);
  const int ntiles = nw->n / 16;
  const int grid = std::max(1, std::min(ntiles, kNumSMs));
  const int per_cta = (ntiles + grid - 1) / grid;
  const size_t tile_bytes = size_t(nw->k / ck) * kChunkBytes;
  const size_t w_total = size_t(ntiles) * tile_bytes;
  if (w_total >= (size_t(1) << 32)) return nx;  // 32-bit offsets
  nx.w = static_cast<const uint8_t*>(nw->w_tf);
  nx.w_stride = uint32_t(per_cta * tile_bytes);
  nx.w_bytes = uint32_t(std::min<size_t>(size_t(kb) * 1024, per_cta * tile_bytes));
  nx.w_total = uint32_t(w_total);
  const size_t srow = nw->fmt == kW4 ? size_t(nw->k / kW4Group) * 2 : (nw->fmt == kINT8 ? 4 : 0);
  if (srow && nw->s) {
    nx.s = static_cast<const uint8_t*>(nw->s);
    nx.s_stride = uint32_t(per_cta * 16 * srow);
    nx.s_bytes = nx.s_stride;
    nx.s_total = uint32_t(size_t(nw->n) * srow);
  }
  nx.ncta = grid;
  return nx;
}

template <int FMT, int PRO, int EPI, int NT, int S>
void launch_tf_s(const LinearW& W, const float* x, int T, const half* gamma, float eps, float* y,
                 cudaStream_t st) {
  const int ntiles = W.n / 16;
  const int grid = std::max(1, std::min(ntiles, kNumSMs));
  const int stage_bytes = S * kChunkBytes;
  const size_t xraw = FMT == kINT8 ? size_t(T) * W.k
                                   : (FMT == kW4 ? size_t(NT) * 4 * W.k + 2 * size_t(NT) * (W.k / kW4Group) * 4
                                                 : size_t(T) * 2 * W.k);
  const size_t xbytes = (xraw + 127) & ~size_t(127);
  const int per_cta = (ntiles + grid - 1) / grid;
  const size_t sbytes = FMT == kW4 ? size_t(per_cta) * 16 * (W.k / kW4Group) * (W.z ? 3 : 2)
                                   : (FMT == kINT8 ? size_t(per_cta) * 16 * 4 : 0);
  const size_t fixed = xbytes + ((sbytes + 127) & ~size_t(127));
  int stages = int((kSmemBudget - std::min<size_t>(fixed, kSmemBudget - 2 * stage_bytes)) / stage_bytes);
  stages = std::max(2, std::min(kMaxStages, stages));
  const size_t smem = fixed + size_t(stages) * stage_bytes;
  if (smem > 200 * 1024) throw ConfigErr("gemv: shared memory budget exceeded");
  static bool attr_done = false;
  if (!attr_done) {
    MSW_CUDA(cudaFuncSetAttribute(gemv_tf_kernel<FMT, PRO, EPI, NT, S>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr_done = true;
  }
  launch_pdl(gemv_tf_kernel<FMT, PRO, EPI, NT, S>, dim3(grid), dim3(kThreads), smem, st,
             static_cast<const uint8_t*>(W.w_tf), W.s, W.n, W.k, x, T, gamma, eps, y, stages,
             t_next, FMT == kW4 ? W.z : static_cast<const uint8_t*>(nullptr));
}

template <int PRO, int EPI, int NT, int S, int GW, bool XREG, bool ZP>
void launch_w4(const LinearW& W, const float* x, int T, const half* gamma, float eps, float* y,
               cudaStream_t st) {
  const int ntiles = W.n / 16;
  const int grid = std::max(1, std::min(ntiles, kNumSMs));
  const int stage_bytes = S * kChunkBytes;
  const int groups = W.k / kW4Group;
  const size_t xbytes = (size_t(NT) * 4 * W.k + (ZP ? 2 : 1) * size_t(NT) * groups * 4 + 127) & ~size_t(127);
  const int per_cta = (ntiles + grid - 1) / grid;
  const size_t sbytes = (size_t(per_cta) * 16 * groups * (W.z ? 3 : 2) + 127) & ~size_t(127);
  const size_t fixed = xbytes + sbytes;
  if (fixed + 2 * size_t(stage_bytes) > size_t(kSmemBudget))
    throw ConfigErr("gemv(w4): shared memory budget exceeded");
  const int stages = std::min<int>(kMaxStages, int((kSmemBudget - fixed) / stage_bytes));
  const size_t smem = fixed + size_t(stages) * stage_bytes;
  static bool attr_done = false;
  if (!attr_done) {
    MSW_CUDA(cudaFuncSetAttribute(gemv_w4_kernel<PRO, EPI, NT, S, GW, XREG, ZP>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr_done = true;
  }
  launch_pdl(gemv_w4_kernel<PRO, EPI, NT, S, GW, XREG, ZP>, dim3(grid), dim3(kThreads), smem, st,
             static_cast<const uint8_t*>(W.w_tf), W.s, W.n, W.k, x, T, gamma, eps, y, stages,
             t_next, W.z);
}

template <int FMT, int PRO, int EPI, int NT>
void launch_tf(const LinearW& W, const float* x, int T, const half* gamma, float eps, float* y,
               cudaStream_t st) {
  const int chunks_tile = W.k / TF<FMT>::kChunkK;
  if constexpr (FMT == kW4 && NT == 1) {  // the GPTQ modes decode batch-1
    static const bool generic = diag_env("MSW_GEMV_W4_GENERIC") != nullptr;  // A/B switch
    if (!generic) {
    if (W.z != nullptr) {  // AWQ zero points
      if (chunks_tile == 64) return launch_w4<PRO, EPI, NT, 64, 1, true, true>(W, x, T, gamma, eps, y, st);
      if (chunks_tile % 64 == 0) return launch_w4<PRO, EPI, NT, 64, 1, false, true>(W, x, T, gamma, eps, y, st);
      if (chunks_tile % 32 == 0 && chunks_tile >= 64)
        return launch_w4<PRO, EPI, NT, 32, 2, false, true>(W, x, T, gamma, eps, y, st);
    } else {
      if (chunks_tile == 64) return launch_w4<PRO, EPI, NT, 64, 1, true, false>(W, x, T, gamma, eps, y, st);
      if (chunks_tile % 64 == 0) return launch_w4<PRO, EPI, NT, 64, 1, false, false>(W, x, T, gamma, eps, y, st);
      if (chunks_tile % 32 == 0 && chunks_tile >= 64)
        return launch_w4<PRO, EPI, NT, 32, 2, false, false>(W, x, T, gamma, eps, y, st);
    }
    }
  }
  if (chunks_tile % 32 == 0) return launch_tf_s<FMT, PRO, EPI, NT, 32>(W, x, T, gamma, eps, y, st);
  if (chunks_tile % 8 == 0) return launch_tf_s<FMT, PRO, EPI, NT, 8>(W, x, T, gamma, eps, y, st);
  if (chunks_tile % 4 == 0) return launch_tf_s<FMT, PRO, EPI, NT, 4>(W, x, T, gamma, eps, y, st);
  throw ConfigErr("gemv: unsupported K for the decode layout");
}

template <int FMT, int NT>
void dispatch_nt(const LinearW& W, int pro, int epi, const float* x, int T, const half* gamma,
                 float eps, float* y, cudaStream_t st) {
#define MSW_GEMV_CASE(P, E) \
  if (pro == P && epi == E) return launch_tf<FMT, P, E, NT>(W, x, T, gamma, eps, y, st);
  MSW_GEMV_CASE(kProPlain, kEpiStore)
  MSW_GEMV_CASE(kProPlain, kEpiResid)
  MSW_GEMV_CASE(kProPlain, kEpiSwiglu)
  MSW_GEMV_CASE(kProNorm, kEpiStore)
  MSW_GEMV_CASE(kProNorm, kEpiResid)
  MSW_GEMV_CASE(kProNorm, kEpiSwiglu)
  if constexpr (FMT == kINT8) {
    MSW_GEMV_CASE(kProPlain, kEpiRaw)
  }
#undef MSW_GEMV_CASE
  throw ConfigErr("gemv: bad prologue/epilogue");
}

template <int FMT>
void dispatch_fmt(const LinearW& W, int pro, int epi, const float* x, int T, const half* gamma,
                  float eps, float* y, cudaStream_t st) {
  if (T == 1) return dispatch_nt<FMT, 1>(W, pro, epi, x, T, gamma, eps, y, st);
  if (T == 2) return dispatch_nt<FMT, 2>(W, pro, epi, x, T, gamma, eps, y, st);
  if (T <= 4) return dispatch_nt<FMT, 4>(W, pro, epi, x, T, gamma, eps, y, st);
  return dispatch_nt<FMT, kGemvMaxTokens>(W, pro, epi, x, T, gamma, eps, y, st);
}

__global__ void gemv_i8_acc_kernel(const int8_t* __restrict__ w, const int8_t* __restrict__ x,
                                   int n, int k, int* __restrict__ acc) {
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= n) return;
  const int nch = k / 16;
  int a = 0;
  for (int c = lane; c < nch; c += 32) {
    const uint4 wv = ld_stream(w + size_t(row) * k + size_t(c) * 16);
    const uint4 xv = *reinterpret_cast<const uint4*>(x + size_t(c) * 16);
    a = __dp4a(int(wv.x), int(xv.x), a);
    a = __dp4a(int(wv.y), int(xv.y), a);
    a = __dp4a(int(wv.z), int(xv.z), a);
    a = __dp4a(int(wv.w), int(xv.w), a);
  }
  a = warp_sum_i(a);
  if (lane == 0) acc[row] = a;
}

}  // namespace

#ifdef MSW_TRACE
extern "C" int msw_trace_set(void* buf) {
  return cudaMemcpyToSymbol(g_msw_trace, &buf, sizeof(buf)) == cudaSuccess ? 0 : 1;
}
#endif

void launch_gemv_(const LinearW& W, int pro, int epi, const float* x, int T, const half* gamma,
                  float eps, float* y, cudaStream_t st);

void launch_gemv(const LinearW& W, int pro, int epi, const float* x, int T, const half* gamma,
                 float eps, float* y, cudaStream_t st, const LinearW* next) {
  t_next = make_l2_next(W.fmt, next);
  try {
    launch_gemv_(W, pro, epi, x, T, gamma, eps, y, st);
  } catch (...) {
    t_next = L2Next();
    throw;
  }
  t_next = L2Next();
}

void launch_gemv_(const LinearW& W, int pro, int epi, const float* x, int T, const half* gamma,
                  float eps, float* y, cudaStream_t st) {
  if (W.n % 16 != 0 || W.k % 128 != 0) throw ConfigErr("gemv: n % 16, k % 128 required");
  if (T < 1 || T > kGemvMaxTokens) throw ConfigErr("gemv: 1..6 tokens");
  if (!W.w_tf) throw ConfigErr("gemv: decode (tile-fragment) weight layout missing");
  switch (W.fmt) {
    case kFP16: return dispatch_fmt<kFP16>(W, pro, epi, x, T, gamma, eps, y, st);
    case kINT8: return dispatch_fmt<kINT8>(W, pro, epi, x, T, gamma, eps, y, st);
    case kW4:
      if (T > 1 && size_t(kGemvMaxTokens) * 4 * W.k > 120 * 1024) {
        // large-K multi-token W4 (not on any engine path: GPTQ modes are batch-1):
        // one launch per token keeps the x staging within shared memory
        for (int t = 0; t < T; ++t)
          dispatch_fmt<kW4>(W, pro, epi, x + size_t(t) * W.k, 1, gamma, eps,
                            y + size_t(t) * (epi == kEpiSwiglu ? W.n / 2 : W.n), st);
        return;
      }
      return dispatch_fmt<kW4>(W, pro, epi, x, T, gamma, eps, y, st);
    default: throw ConfigErr("gemv: bad weight format");
  }
}

size_t tf_bytes(int fmt, int n, int k) {
  return fmt == kFP16 ? size_t(n) * k * 2 : (fmt == kINT8 ? size_t(n) * k : size_t(n) * k / 2);
}

void launch_repack_tf(int fmt, const void* src, int n, int k, void* dst, cudaStream_t st) {
  if (n % 16 || k % 128) throw ConfigErr("repack_tf: n % 16, k % 128 required");
  repack_tf_kernel<<<kNumSMs * 8, 256, 0, st>>>(fmt, static_cast<const uint8_t*>(src), n, k,
                                                static_cast<uint8_t*>(dst));
  MSW_LAUNCH_CHECK();
}

void launch_gemv_i8_acc(const int8_t* w, const int8_t* x, int n, int k, int* acc, cudaStream_t st) {
  if (k % 16 != 0) throw ConfigErr("gemv_i8_acc: k must be a multiple of 16");
  gemv_i8_acc_kernel<<<ceil_div(n, 8), 256, 0, st>>>(w, x, n, k, acc);
  MSW_LAUNCH_CHECK();
}

}  // namespace msw
