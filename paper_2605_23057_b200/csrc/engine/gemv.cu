// Decode GEMV (1..6 tokens) for the three weight formats, TMA-fed, on the
// tensor cores.
//
// HBM-bound: every weight byte is read once per step. Decode weights are
// stored "tile-fragment" (TF): 16-row tiles, each a contiguous run of 512-byte
// chunks, a chunk being one 16-byte mma.sync A fragment per lane:
//   FP16 : m16n8k16 f16 -> f32, chunk = 16 rows x 16 k
//   INT8 : m16n8k32 s8 -> s32 (exact), chunk = 16 rows x 32 k
//   W4   : m16n8k16 f16 on lop3/hsub2-dequantised (q-8), chunk = 16 rows x 64 k
//          (4 k16 steps), group scale applied in fp32 per 128 k
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

namespace msw {
namespace {

constexpr int kConsumers = 8;
constexpr int kThreads = (kConsumers + 1) * 32;  // + producer warp
constexpr int kConsThreads = kConsumers * 32;
constexpr int kChunkBytes = 512;
constexpr int kMaxStages = 8;
constexpr int kSmemBudget = 200 * 1024;

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

template <int FMT>
struct TF {
  static constexpr int kChunkK = FMT == kFP16 ? 16 : (FMT == kINT8 ? 32 : 64);
  static constexpr int kMinChunksPerWarp = FMT == kW4 ? 2 : 1;  // a W4 scale group is 2 chunks
};

// Stage size in chunks: the largest power of two <= 32 dividing a tile's chunks.
__host__ __device__ inline int stage_chunks(int chunks_per_tile) {
  int s = 32;
  while (s > 1 && chunks_per_tile % s) s >>= 1;
  return s;
}

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

// x fp32 [T, k] -> smem: fp16 [NT][k] (FP16 / W4) or int8 [NT][k] + scale.
template <int FMT, int PRO, int NT>
__device__ __forceinline__ void prologue(const float* __restrict__ x, const half* __restrict__ gamma,
                                         float eps, int k, int T, uint8_t* xs, float* red,
                                         float* xscale) {
  const int tid = threadIdx.x;
  for (int t = 0; t < NT; ++t) {
    const int bytes = FMT == kINT8 ? k : 2 * k;
    if (t >= T) {
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
      char4* xq = reinterpret_cast<char4*>(xs + size_t(t) * k);
      auto q = [&](float v) -> signed char {
        const float u = amax > 0.0f ? rintf(v / s) : 0.0f;
        return static_cast<signed char>(fminf(fmaxf(u, -127.0f), 127.0f));
      };
      for (int i = tid; i < k4; i += kConsThreads) {
        const float4 v = act4(i);
        xq[i] = make_char4(q(v.x), q(v.y), q(v.z), q(v.w));
      }
      if (tid == 0) xscale[t] = s;
    } else {
      half2* xh = reinterpret_cast<half2*>(xs + size_t(t) * 2 * k);
      for (int i = tid; i < k4; i += kConsThreads) {
        const float4 v = act4(i);
        xh[2 * i] = __floats2half2_rn(v.x, v.y);
        xh[2 * i + 1] = __floats2half2_rn(v.z, v.w);
      }
    }
    named_sync(1, kConsThreads);
  }
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

template <int FMT, int PRO, int EPI, int NT>
__global__ void __launch_bounds__(kThreads, 1)
    gemv_tf_kernel(const uint8_t* __restrict__ wtf, const void* __restrict__ ws, int n, int k,
                   const float* __restrict__ x, int T, const half* __restrict__ gamma, float eps,
                   float* __restrict__ y, int n_stages) {
  using Acc = typename std::conditional<FMT == kINT8, int, float>::type;
  constexpr int CK = TF<FMT>::kChunkK;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full[kMaxStages], empty[kMaxStages];
  __shared__ float red[32];
  __shared__ float xscale[NT];
  __shared__ uint32_t part[kConsumers][16][8];  // raw 32-bit partials (f32 or s32)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int chunks_tile = k / CK;
  const int S = stage_chunks(chunks_tile);  // chunks per stage
  const int cpw = max(S / kConsumers, TF<FMT>::kMinChunksPerWarp);
  const int active_warps = S / cpw;
  const int ntiles = n / 16;
  const int per_cta = (ntiles + gridDim.x - 1) / gridDim.x;
  const int tile_begin = blockIdx.x * per_cta;
  const int tile_end = min(ntiles, tile_begin + per_cta);
  const int stages_tile = chunks_tile / S;
  const int total_stages = tile_end > tile_begin ? (tile_end - tile_begin) * stages_tile : 0;
  const int stage_bytes = S * kChunkBytes;
  const int xbytes = NT * (FMT == kINT8 ? k : 2 * k);
  uint8_t* xs = smem;
  uint8_t* ring = smem + ((xbytes + 127) & ~127);

  if (threadIdx.x == 0) {
    for (int s = 0; s < n_stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], active_warps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kConsumers) {
    // producer: stream this CTA's contiguous weight range. Weights only, so it
    // runs ahead of griddepcontrol.wait and fills the ring during the
    // previous kernel.
    if (lane == 0) {
      const uint8_t* src = wtf + size_t(tile_begin) * chunks_tile * kChunkBytes;
      for (int st = 0; st < total_stages; ++st) {
        const int s = st % n_stages;
        mbar_wait(&empty[s], ((st / n_stages) & 1) ^ 1);
        mbar_expect_tx(&full[s], stage_bytes);
        bulk_g2s(ring + size_t(s) * stage_bytes, src + size_t(st) * stage_bytes, stage_bytes,
                 &full[s]);
      }
    }
    pdl_wait();
    pdl_trigger();
    return;
  }

  // consumers
  pdl_wait();
  pdl_trigger();
  prologue<FMT, PRO, NT>(x, gamma, eps, k, T, xs, red, xscale);
  const int g = lane >> 2, tq = lane & 3;
  const bool has_tok = g < T;  // this lane's MMA column is a real token
  const int groups_k = k / kW4Group;
  const half2 k1032 = __float2half2_rn(1032.0f);

  Acc acc[4] = {0, 0, 0, 0};
  float cg[4] = {0.f, 0.f, 0.f, 0.f};  // W4: current 128-k group
  for (int st = 0; st < total_stages; ++st) {
    const int s = st % n_stages;
    const int tile = tile_begin + st / stages_tile;
    const int c_tile0 = (st % stages_tile) * S;  // first chunk (within the tile) of the stage
    mbar_wait(&full[s], (st / n_stages) & 1);
    if (warp < active_warps) {
      const uint4* stage = reinterpret_cast<const uint4*>(ring + size_t(s) * stage_bytes);
#pragma unroll 2
      for (int j = 0; j < cpw; ++j) {
        const int c_local = warp * cpw + j;
        const int c = c_tile0 + c_local;  // chunk index within the tile
        const uint4 a4 = stage[c_local * 32 + lane];
        if (FMT == kFP16) {
          const int kk = c * 16 + 2 * tq;
          uint32_t b0 = 0, b1 = 0;
          if (has_tok) {
            const half* xr = reinterpret_cast<const half*>(xs) + size_t(g) * k;
            b0 = *reinterpret_cast<const uint32_t*>(xr + kk);
            b1 = *reinterpret_cast<const uint32_t*>(xr + kk + 8);
          }
          const uint32_t a[4] = {a4.x, a4.y, a4.z, a4.w};
          mma_f16(reinterpret_cast<float(&)[4]>(acc), a, b0, b1);
        } else if (FMT == kINT8) {
          const int kk = c * 32 + 4 * tq;
          uint32_t b0 = 0, b1 = 0;
          if (has_tok) {
            const int8_t* xr = reinterpret_cast<const int8_t*>(xs) + size_t(g) * k;
            b0 = *reinterpret_cast<const uint32_t*>(xr + kk);
            b1 = *reinterpret_cast<const uint32_t*>(xr + kk + 16);
          }
          const uint32_t a[4] = {a4.x, a4.y, a4.z, a4.w};
          mma_s8(reinterpret_cast<int(&)[4]>(acc), a, b0, b1);
        } else {
          const uint32_t wv[4] = {a4.x, a4.y, a4.z, a4.w};
          const half* xr = reinterpret_cast<const half*>(xs) + size_t(g) * k;
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const int kk = c * 64 + jj * 16 + 2 * tq;
            uint32_t b0 = 0, b1 = 0;
            if (has_tok) {
              b0 = *reinterpret_cast<const uint32_t*>(xr + kk);
              b1 = *reinterpret_cast<const uint32_t*>(xr + kk + 8);
            }
            uint32_t a[4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
              a[i] = h22u(__hsub2(u2h2(lop3_and_or(wv[jj] >> (4 * i), 0x000F000Fu, 0x64006400u)),
                                  k1032));
            mma_f16(cg, a, b0, b1);
          }
          if (c & 1) {  // end of a 128-k group: fp32 group scale per row
            const half* sc = static_cast<const half*>(ws);
            const int grp = c >> 1;
            const float slo = __half2float(sc[size_t(tile * 16 + g) * groups_k + grp]);
            const float shi = __half2float(sc[size_t(tile * 16 + g + 8) * groups_k + grp]);
            acc[0] = fmaf(slo, cg[0], acc[0]);
            acc[1] = fmaf(slo, cg[1], acc[1]);
            acc[2] = fmaf(shi, cg[2], acc[2]);
            acc[3] = fmaf(shi, cg[3], acc[3]);
            cg[0] = cg[1] = cg[2] = cg[3] = 0.f;
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if ((st + 1) % stages_tile == 0) {
      // tile complete: reduce the 16 x 8 partials of all warps, fused epilogue
      uint32_t raw[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (FMT == kINT8) raw[i] = warp < active_warps ? uint32_t(int(acc[i])) : 0u;
        else raw[i] = __float_as_uint(warp < active_warps ? float(acc[i]) : 0.0f);
      }
      part[warp][g][2 * tq] = raw[0];
      part[warp][g][2 * tq + 1] = raw[1];
      part[warp][g + 8][2 * tq] = raw[2];
      part[warp][g + 8][2 * tq + 1] = raw[3];
      named_sync(1, kConsThreads);
      if (threadIdx.x < 128) {
        const int row = threadIdx.x >> 3, col = threadIdx.x & 7;
        float v;
        if (FMT == kINT8) {
          int iv = 0;  // exact int32 across warps
#pragma unroll
          for (int w2 = 0; w2 < kConsumers; ++w2) iv += int(part[w2][row][col]);
          v = float(iv);
        } else {
          v = 0.f;
#pragma unroll
          for (int w2 = 0; w2 < kConsumers; ++w2) v += __uint_as_float(part[w2][row][col]);
        }
        const float vn = __shfl_down_sync(0xffffffffu, v, 8);  // row + 1, same column
        if ((row & 1) == 0 && col < T) {
          float v0 = v, v1 = vn;
          if (FMT == kINT8) {
            const float* sw = static_cast<const float*>(ws);
            v0 = (v0 * xscale[col]) * sw[tile * 16 + row];
            v1 = (v1 * xscale[col]) * sw[tile * 16 + row + 1];
          }
          store_pair<EPI>(y, n, col, tile * 16 + row, v0, v1);
        }
      }
      named_sync(1, kConsThreads);
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i] = 0;
    }
  }
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
      // element e of the k16 step: pair e>>1 -> a0..a3, e&1 -> first/second k
      const uint32_t* sw = reinterpret_cast<const uint32_t*>(src);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int pr = e >> 1, hi = e & 1;
        const int row = tile * 16 + g + ((pr & 1) ? 8 : 0);
        const int kk = c * 64 + reg * 16 + 2 * tq + ((pr & 2) ? 8 : 0) + hi;
        const uint32_t w = sw[size_t(row) * (k / 8) + kk / 8];
        const int si = kk & 7;
        const uint32_t q = (w >> (4 * ((si >> 1) + 4 * (si & 1)))) & 0xF;
        word |= q << (4 * ((e >> 1) + 4 * (e & 1)));
      }
    }
    reinterpret_cast<uint32_t*>(dst)[i] = word;
  }
}

template <int FMT, int PRO, int EPI, int NT>
void launch_tf(const LinearW& W, const float* x, int T, const half* gamma, float eps, float* y,
               cudaStream_t st) {
  const int ntiles = W.n / 16;
  const int grid = std::max(1, std::min(ntiles, kNumSMs));
  const int chunks_tile = W.k / TF<FMT>::kChunkK;
  const int stage_bytes = stage_chunks(chunks_tile) * kChunkBytes;
  const size_t xbytes = (size_t(NT) * (FMT == kINT8 ? W.k : 2 * W.k) + 127) & ~size_t(127);
  int stages = int((kSmemBudget - std::min<size_t>(xbytes, kSmemBudget - 2 * stage_bytes)) / stage_bytes);
  stages = std::max(2, std::min(kMaxStages, stages));
  const size_t smem = xbytes + size_t(stages) * stage_bytes;
  static bool attr_done = false;
  if (!attr_done) {
    MSW_CUDA(cudaFuncSetAttribute(gemv_tf_kernel<FMT, PRO, EPI, NT>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr_done = true;
  }
  launch_pdl(gemv_tf_kernel<FMT, PRO, EPI, NT>, dim3(grid), dim3(kThreads), smem, st,
             static_cast<const uint8_t*>(W.w_tf), W.s, W.n, W.k, x, T, gamma, eps, y, stages);
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

void launch_gemv(const LinearW& W, int pro, int epi, const float* x, int T, const half* gamma,
                 float eps, float* y, cudaStream_t st) {
  if (W.n % 16 != 0 || W.k % 128 != 0) throw ConfigErr("gemv: n % 16, k % 128 required");
  if (T < 1 || T > kGemvMaxTokens) throw ConfigErr("gemv: 1..6 tokens");
  if (!W.w_tf) throw ConfigErr("gemv: decode (tile-fragment) weight layout missing");
  switch (W.fmt) {
    case kFP16: return dispatch_fmt<kFP16>(W, pro, epi, x, T, gamma, eps, y, st);
    case kINT8: return dispatch_fmt<kINT8>(W, pro, epi, x, T, gamma, eps, y, st);
    case kW4: return dispatch_fmt<kW4>(W, pro, epi, x, T, gamma, eps, y, st);
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
