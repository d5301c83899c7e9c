// Decode GEMV (1..6 tokens) for the three weight formats.
//
// HBM-bound: every weight byte is read once per step with 128-bit
// ld.global.nc.L1::no_allocate loads, coalesced across the warp.
//
//  * FP16 / W8A8 (CUDA cores): one warp owns a PAIR of output rows (so the
//    SwiGLU epilogue combines gate/up, interleaved rows 2i / 2i+1, in
//    registers), lanes stride 16-byte chunks along K, warp-shuffle reduction;
//    W8A8 uses dp4a with exact int32 accumulation.
//  * W4 g128 (tensor cores, mma.sync m16n8k16): weights are stored in the
//    fragment order of the A operand, so one 16-byte load per lane is four
//    k16 steps of a 16-row tile; dequant is lop3 (nibble -> fp16 1024+q) and
//    one hsub2 -> (q-8) exact; the group scale is applied in fp32 per 128-k
//    group. The 8 MMA columns are up to 8 tokens (verify / tiny batches) for
//    free. K is split across the 8 warps of a CTA and reduced in smem.
//
// Grids are persistent (<= 2 CTAs per SM), so the activation prologue
// (RMSNorm + fp16 rounding or per-token int8 quantisation, into smem) runs
// once per CTA, and every kernel is launched with programmatic dependent
// launch: the first weight loads are issued BEFORE griddepcontrol.wait, so
// they overlap the previous kernel's tail.
#include "kernels.cuh"

namespace msw {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kUnroll = 4;      // 16-byte chunks per lane per row in flight (CUDA-core path)
constexpr int kCtasPerSm = 2;

__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ half2 u2h2(uint32_t u) { return *reinterpret_cast<half2*>(&u); }
__device__ __forceinline__ uint32_t h22u(half2 h) { return *reinterpret_cast<uint32_t*>(&h); }

// ---------------------------------------------------------------- prologue
// x fp32 [T, k] -> smem: fp16 [NT][k] (FP16 / W4) or int8 [NT][k] + scale.
template <int FMT, int PRO, int NT>
__device__ __forceinline__ void prologue(const float* __restrict__ x, const half* __restrict__ gamma,
                                         float eps, int k, int T, uint8_t* smem, float* red,
                                         float* xscale) {
  for (int t = 0; t < NT; ++t) {
    if (t >= T) {  // padding token
      const int bytes = FMT == kINT8 ? k : 2 * k;
      for (int i = threadIdx.x; i < bytes / 16; i += kThreads)
        reinterpret_cast<uint4*>(smem + size_t(t) * bytes)[i] = make_uint4(0, 0, 0, 0);
      if (threadIdx.x == 0) xscale[t] = 0.0f;
      continue;
    }
    const float4* xt = reinterpret_cast<const float4*>(x + size_t(t) * k);
    const int k4 = k / 4;
    float r = 1.0f;
    if (PRO == kProNorm) {
      float ss = 0.0f;
      for (int i = threadIdx.x; i < k4; i += kThreads) {
        const float4 v = xt[i];
        ss = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, ss))));
      }
      ss = block_sum(ss, red);
      r = 1.0f / sqrtf(ss / float(k) + eps);
    }
    auto act4 = [&](int i) -> float4 {
      float4 v = xt[i];
      if (PRO == kProNorm) {
        const half2* g = reinterpret_cast<const half2*>(gamma) + 2 * i;
        const float2 g0 = __half22float2(g[0]), g1 = __half22float2(g[1]);
        v.x = (v.x * r) * g0.x;
        v.y = (v.y * r) * g0.y;
        v.z = (v.z * r) * g1.x;
        v.w = (v.w * r) * g1.y;
      }
      return v;
    };
    if (FMT == kINT8) {
      float amax = 0.0f;
      for (int i = threadIdx.x; i < k4; i += kThreads) {
        const float4 v = act4(i);
        amax = fmaxf(amax, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
      }
      amax = block_max(amax, red);
      const float s = amax / 127.0f;
      char4* xq = reinterpret_cast<char4*>(smem + size_t(t) * k);
      auto q = [&](float v) -> signed char {
        const float u = amax > 0.0f ? rintf(v / s) : 0.0f;
        return static_cast<signed char>(fminf(fmaxf(u, -127.0f), 127.0f));
      };
      for (int i = threadIdx.x; i < k4; i += kThreads) {
        const float4 v = act4(i);
        xq[i] = make_char4(q(v.x), q(v.y), q(v.z), q(v.w));
      }
      if (threadIdx.x == 0) xscale[t] = s;
    } else {
      half2* xh = reinterpret_cast<half2*>(smem + size_t(t) * 2 * k);
      for (int i = threadIdx.x; i < k4; i += kThreads) {
        const float4 v = act4(i);
        xh[2 * i] = __floats2half2_rn(v.x, v.y);
        xh[2 * i + 1] = __floats2half2_rn(v.z, v.w);
      }
    }
    __syncthreads();
  }
  __syncthreads();
}

template <int EPI>
__device__ __forceinline__ void store_out(float* y, int n, int t, int row, float v0, float v1) {
  // rows (row, row+1): STORE / RESID write both; SWIGLU writes silu(v0) * v1 at row/2
  if (EPI == kEpiStore) {
    y[size_t(t) * n + row] = v0;
    y[size_t(t) * n + row + 1] = v1;
  } else if (EPI == kEpiResid) {
    y[size_t(t) * n + row] += v0;
    y[size_t(t) * n + row + 1] += v1;
  } else {
    y[size_t(t) * (n / 2) + row / 2] = silu(v0) * v1;
  }
}

// ------------------------------------------------- FP16 / W8A8 (CUDA cores)
template <int FMT, int PRO, int EPI, int NT>
__global__ void __launch_bounds__(kThreads) gemv_cc_kernel(const uint8_t* __restrict__ w,
                                                           const void* __restrict__ ws, int n, int k,
                                                           const float* __restrict__ x, int T,
                                                           const half* __restrict__ gamma,
                                                           float eps, float* __restrict__ y) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ float red[32];
  __shared__ float xscale[NT];
  using Acc = typename std::conditional<FMT == kINT8, int, float>::type;
  constexpr int E = FMT == kINT8 ? 16 : 8;  // elements per 16-byte chunk
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nch = k / E;
  const size_t row_bytes = size_t(nch) * 16;
  const int tok16 = (FMT == kINT8 ? k : 2 * k) / 16;  // uint4 per token in smem
  const int npairs = n >> 1;
  const int groups = (nch + 32 * kUnroll - 1) / (32 * kUnroll);
  const int pair_stride = gridDim.x * kWarps;
  int pair = blockIdx.x * kWarps + warp;

  uint4 buf[2][kUnroll];
  auto load = [&](int p, int g, uint4 (&b)[2][kUnroll]) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const uint8_t* row = w + size_t(2 * p + r) * row_bytes;
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int c = (g * kUnroll + u) * 32 + lane;
        b[r][u] = c < nch ? ld_stream(row + size_t(c) * 16) : make_uint4(0, 0, 0, 0);
      }
    }
  };
  if (pair < npairs) load(pair, 0, buf);  // weights only: safe before the dependency wait
  pdl_wait();
  pdl_trigger();
  prologue<FMT, PRO, NT>(x, gamma, eps, k, T, smem, red, xscale);
  const uint4* xs = reinterpret_cast<const uint4*>(smem);

  for (; pair < npairs; pair += pair_stride) {
    Acc acc0[NT], acc1[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) acc0[t] = acc1[t] = 0;
    for (int g = 0; g < groups; ++g) {
      uint4 nxt[2][kUnroll];
      if (g + 1 < groups) load(pair, g + 1, nxt);
      else if (pair + pair_stride < npairs) load(pair + pair_stride, 0, nxt);
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int c = (g * kUnroll + u) * 32 + lane;
        if (c < nch) {
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            const uint4 xv = xs[t * tok16 + c];  // one smem load serves both rows
            if (FMT == kINT8) {
              acc0[t] = __dp4a(int(buf[0][u].x), int(xv.x), acc0[t]);
              acc0[t] = __dp4a(int(buf[0][u].y), int(xv.y), acc0[t]);
              acc0[t] = __dp4a(int(buf[0][u].z), int(xv.z), acc0[t]);
              acc0[t] = __dp4a(int(buf[0][u].w), int(xv.w), acc0[t]);
              acc1[t] = __dp4a(int(buf[1][u].x), int(xv.x), acc1[t]);
              acc1[t] = __dp4a(int(buf[1][u].y), int(xv.y), acc1[t]);
              acc1[t] = __dp4a(int(buf[1][u].z), int(xv.z), acc1[t]);
              acc1[t] = __dp4a(int(buf[1][u].w), int(xv.w), acc1[t]);
            } else {
              const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
              const uint32_t w0[4] = {buf[0][u].x, buf[0][u].y, buf[0][u].z, buf[0][u].w};
              const uint32_t w1[4] = {buf[1][u].x, buf[1][u].y, buf[1][u].z, buf[1][u].w};
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float2 b = __half22float2(u2h2(xw[i]));
                const float2 a0 = __half22float2(u2h2(w0[i]));
                const float2 a1 = __half22float2(u2h2(w1[i]));
                acc0[t] = fmaf(a0.x, b.x, fmaf(a0.y, b.y, acc0[t]));
                acc1[t] = fmaf(a1.x, b.x, fmaf(a1.y, b.y, acc1[t]));
              }
            }
          }
        }
      }
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) buf[r][u] = nxt[r][u];
    }
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      float v0, v1;
      if (FMT == kINT8) {
        const int a0 = warp_sum_i(int(acc0[t])), a1 = warp_sum_i(int(acc1[t]));
        const float* sw = static_cast<const float*>(ws);
        v0 = (float(a0) * xscale[t]) * sw[2 * pair];
        v1 = (float(a1) * xscale[t]) * sw[2 * pair + 1];
      } else {
        v0 = warp_sum(float(acc0[t]));
        v1 = warp_sum(float(acc1[t]));
      }
      if (lane == 0 && t < T) store_out<EPI>(y, n, t, 2 * pair, v0, v1);
    }
  }
}

// ------------------------------------------------------- W4 (mma.sync path)
// Layout "mma4": [n/16 row tiles][k/64 chunks][32 lanes][4 words]; word j =
// k16 step j of the chunk; its 8 nibbles (position (i>>1) + 4*(i&1) for
// element i) are the A fragment a0..a3 of lane (g = lane/4, t = lane%4):
// a0 = (row g, k 2t..2t+1), a1 = (row g+8, k 2t..), a2 = (row g, k 2t+8..),
// a3 = (row g+8, k 2t+8..).
constexpr int kW4Unroll = 8;  // chunks (512 B per warp) in flight per warp

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int PRO, int EPI, int NT>
__global__ void __launch_bounds__(kThreads) gemv_w4_kernel(const uint4* __restrict__ wq,
                                                           const half* __restrict__ ws, int n, int k,
                                                           const float* __restrict__ x, int T,
                                                           const half* __restrict__ gamma,
                                                           float eps, float* __restrict__ y) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ float red[32];
  __shared__ float xscale[NT];
  __shared__ float part[kWarps][16][8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int nchunks = k / 64;
  // K slice of this warp, in chunks; even so a 128-k scale group never straddles warps
  const int per_warp = (((nchunks + kWarps - 1) / kWarps) + 1) & ~1;
  const int c_begin = warp * per_warp;
  const int c_end = min(nchunks, c_begin + per_warp);
  const int ntiles = n / 16;
  const int groups_k = k / kW4Group;
  int tile = blockIdx.x;

  uint4 cur[kW4Unroll];
  auto load = [&](int tl, int c0, uint4 (&b)[kW4Unroll]) {
    const uint4* base = wq + (size_t(tl) * nchunks) * 32 + lane;
#pragma unroll
    for (int u = 0; u < kW4Unroll; ++u) {
      const int c = c0 + u;
      b[u] = c < c_end ? ld_stream(base + size_t(c) * 32) : make_uint4(0, 0, 0, 0);
    }
  };
  if (tile < ntiles) load(tile, c_begin, cur);
  pdl_wait();
  pdl_trigger();
  prologue<kW4, PRO, NT>(x, gamma, eps, k, T, smem, red, xscale);
  const half* xs = reinterpret_cast<const half*>(smem);
  const half2 k1032 = __float2half2_rn(1032.0f);
  const bool has_tok = g < NT && g < T;

  for (; tile < ntiles; tile += gridDim.x) {
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    float cg[4] = {0.f, 0.f, 0.f, 0.f};
    const half* s_lo = ws + size_t(tile * 16 + g) * groups_k;
    const half* s_hi = ws + size_t(tile * 16 + g + 8) * groups_k;
    for (int c0 = c_begin; c0 < c_end; c0 += kW4Unroll) {
      uint4 nxt[kW4Unroll];
      if (c0 + kW4Unroll < c_end) load(tile, c0 + kW4Unroll, nxt);
      else if (tile + int(gridDim.x) < ntiles) load(tile + gridDim.x, c_begin, nxt);
#pragma unroll
      for (int u = 0; u < kW4Unroll; ++u) {
        const int c = c0 + u;
        if (c < c_end) {
          const uint32_t wv[4] = {cur[u].x, cur[u].y, cur[u].z, cur[u].w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int kk = c * 64 + j * 16 + 2 * tq;
            uint32_t b0 = 0, b1 = 0;
            if (has_tok) {
              b0 = *reinterpret_cast<const uint32_t*>(xs + size_t(g) * k + kk);
              b1 = *reinterpret_cast<const uint32_t*>(xs + size_t(g) * k + kk + 8);
            }
            uint32_t a[4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
              a[i] = h22u(__hsub2(u2h2(lop3_and_or(wv[j] >> (4 * i), 0x000F000Fu, 0x64006400u)), k1032));
            mma16816(cg, a, b0, b1);
          }
          if (c & 1) {  // end of a 128-k group: apply the fp32 group scale
            const int grp = c >> 1;
            const float slo = __half2float(s_lo[grp]), shi = __half2float(s_hi[grp]);
            acc[0] = fmaf(slo, cg[0], acc[0]);
            acc[1] = fmaf(slo, cg[1], acc[1]);
            acc[2] = fmaf(shi, cg[2], acc[2]);
            acc[3] = fmaf(shi, cg[3], acc[3]);
            cg[0] = cg[1] = cg[2] = cg[3] = 0.f;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kW4Unroll; ++u) cur[u] = nxt[u];
    }
    // cross-warp K reduction: lane holds (row g, cols 2tq, 2tq+1) and (row g+8, ...)
    part[warp][g][2 * tq] = acc[0];
    part[warp][g][2 * tq + 1] = acc[1];
    part[warp][g + 8][2 * tq] = acc[2];
    part[warp][g + 8][2 * tq + 1] = acc[3];
    __syncthreads();
    if (threadIdx.x < 128) {
      const int row = threadIdx.x >> 3, col = threadIdx.x & 7;
      float v = 0.f;
#pragma unroll
      for (int w2 = 0; w2 < kWarps; ++w2) v += part[w2][row][col];
      const float v_next = __shfl_down_sync(0xffffffffu, v, 8);  // row + 1, same column
      if ((row & 1) == 0 && col < T) store_out<EPI>(y, n, col, tile * 16 + row, v, v_next);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------- launchers
template <int FMT, int PRO, int EPI, int NT>
void launch_cc(const LinearW& W, const float* x, int T, const half* gamma, float eps, float* y,
               cudaStream_t st) {
  const int npairs = W.n / 2;
  const int grid = std::max(1, std::min(ceil_div(npairs, kWarps), kNumSMs * kCtasPerSm));
  const size_t smem = size_t(NT) * (FMT == kINT8 ? size_t(W.k) : size_t(W.k) * 2);
  static bool attr_done = false;
  if (!attr_done) {
    MSW_CUDA(cudaFuncSetAttribute(gemv_cc_kernel<FMT, PRO, EPI, NT>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr_done = true;
  }
  launch_pdl(gemv_cc_kernel<FMT, PRO, EPI, NT>, dim3(grid), dim3(kThreads), smem, st,
             static_cast<const uint8_t*>(W.w), W.s, W.n, W.k, x, T, gamma, eps, y);
}

template <int PRO, int EPI, int NT>
void launch_w4(const LinearW& W, const float* x, int T, const half* gamma, float eps, float* y,
               cudaStream_t st) {
  const int grid = std::max(1, std::min(W.n / 16, kNumSMs * kCtasPerSm));
  const size_t smem = size_t(NT) * size_t(W.k) * 2;
  static bool attr_done = false;
  if (!attr_done) {
    MSW_CUDA(cudaFuncSetAttribute(gemv_w4_kernel<PRO, EPI, NT>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr_done = true;
  }
  launch_pdl(gemv_w4_kernel<PRO, EPI, NT>, dim3(grid), dim3(kThreads), smem, st,
             static_cast<const uint4*>(W.w_mma), static_cast<const half*>(W.s), W.n, W.k, x, T,
             gamma, eps, y);
}

template <int FMT, int NT>
void dispatch_nt(const LinearW& W, int pro, int epi, const float* x, int T, const half* gamma,
                 float eps, float* y, cudaStream_t st) {
#define MSW_GEMV_CASE(P, E)                                                  \
  if (pro == P && epi == E) {                                                \
    if (FMT == kW4) return launch_w4<P, E, NT>(W, x, T, gamma, eps, y, st);  \
    return launch_cc<FMT == kW4 ? kFP16 : FMT, P, E, NT>(W, x, T, gamma, eps, y, st); \
  }
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
  const int row = blockIdx.x * kWarps + (threadIdx.x >> 5);
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

// row-packed W4 ([n][k/8] words, nibble position (i>>1)+4(i&1)) -> mma4 layout
__global__ void repack_w4_mma_kernel(const uint32_t* __restrict__ src, int n, int k,
                                     uint32_t* __restrict__ dst) {
  const int nchunks = k / 64;
  const long long total = (long long)(n / 16) * nchunks * 32 * 4;  // words
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int j = int(i & 3);
    const int lane = int((i >> 2) & 31);
    const long long tc = i >> 7;
    const int c = int(tc % nchunks);
    const int tile = int(tc / nchunks);
    const int g = lane >> 2, tq = lane & 3;
    uint32_t word = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) {  // element e of the A fragment
      const int pair = e >> 1, hi = e & 1;
      const int row = tile * 16 + g + ((pair & 1) ? 8 : 0);
      const int kk = c * 64 + j * 16 + 2 * tq + ((pair & 2) ? 8 : 0) + hi;
      const uint32_t sw = src[size_t(row) * (k / 8) + kk / 8];
      const int si = kk & 7;
      const uint32_t q = (sw >> (4 * ((si >> 1) + 4 * (si & 1)))) & 0xF;
      word |= q << (4 * ((e >> 1) + 4 * (e & 1)));
    }
    dst[i] = word;
  }
}

}  // namespace

void launch_gemv(const LinearW& W, int pro, int epi, const float* x, int T, const half* gamma,
                 float eps, float* y, cudaStream_t st) {
  if (W.n % 16 != 0 || W.k % 128 != 0) throw ConfigErr("gemv: n % 16, k % 128 required");
  if (T < 1 || T > kGemvMaxTokens) throw ConfigErr("gemv: 1..6 tokens");
  switch (W.fmt) {
    case kFP16: return dispatch_fmt<kFP16>(W, pro, epi, x, T, gamma, eps, y, st);
    case kINT8: return dispatch_fmt<kINT8>(W, pro, epi, x, T, gamma, eps, y, st);
    case kW4:
      if (!W.w_mma) throw ConfigErr("gemv: W4 needs the mma4 layout");
      return dispatch_fmt<kW4>(W, pro, epi, x, T, gamma, eps, y, st);
    default: throw ConfigErr("gemv: bad weight format");
  }
}

void launch_repack_w4_mma(const uint32_t* packed, int n, int k, uint32_t* mma4, cudaStream_t st) {
  if (n % 16 || k % 128) throw ConfigErr("repack_w4: n % 16, k % 128 required");
  repack_w4_mma_kernel<<<kNumSMs * 8, 256, 0, st>>>(packed, n, k, mma4);
  MSW_LAUNCH_CHECK();
}

void launch_gemv_i8_acc(const int8_t* w, const int8_t* x, int n, int k, int* acc, cudaStream_t st) {
  if (k % 16 != 0) throw ConfigErr("gemv_i8_acc: k must be a multiple of 16");
  gemv_i8_acc_kernel<<<ceil_div(n, kWarps), kThreads, 0, st>>>(w, x, n, k, acc);
  MSW_LAUNCH_CHECK();
}

}  // namespace msw
