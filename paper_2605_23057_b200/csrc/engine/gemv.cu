// Batch-1 decode GEMV for the three weight formats (FP16, W8A8, W4 g128).
//
// HBM-bound: every weight byte is read exactly once per token with
// ld.global.nc.L1::no_allocate 128-bit loads, coalesced across the warp (lane
// l reads 16-byte chunk l, l+32, ...). One warp owns a PAIR of output rows so
// the SwiGLU epilogue can combine gate/up (interleaved rows 2i, 2i+1) without
// leaving registers; the two rows also double the loads in flight. Rows are
// reduced with warp shuffles (no shared-memory reduction, no atomics).
//
// The activation prologue (optional RMSNorm, then fp16 rounding or per-token
// int8 quantisation) runs in every CTA from L2 into shared memory; the first
// weight chunks are issued BEFORE it so the prologue hides under HBM latency.
#include "kernels.cuh"

namespace msw {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kUnroll = 4;  // 16-byte chunks per lane per row in flight

template <int FMT>
struct Fmt;
template <>
struct Fmt<kFP16> {
  static constexpr int kElemsPerChunk = 8;
};
template <>
struct Fmt<kINT8> {
  static constexpr int kElemsPerChunk = 16;
};
template <>
struct Fmt<kW4> {
  static constexpr int kElemsPerChunk = 32;
};

__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

__device__ __forceinline__ half2 u2h2(uint32_t u) { return *reinterpret_cast<half2*>(&u); }

// Dot of one 16-byte weight chunk with the matching activations.
template <int FMT>
struct ChunkDot;

template <>
struct ChunkDot<kFP16> {
  using Acc = float;
  __device__ __forceinline__ static void run(const uint4& w, const uint4* xs, int c, int /*nch*/,
                                             const half2& /*s2*/, float& acc) {
    const uint4 xv = xs[c];
    const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
    const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 a = __half22float2(u2h2(wv[i]));
      const float2 b = __half22float2(u2h2(xw[i]));
      acc = fmaf(a.x, b.x, acc);
      acc = fmaf(a.y, b.y, acc);
    }
  }
};

template <>
struct ChunkDot<kINT8> {
  using Acc = int;
  __device__ __forceinline__ static void run(const uint4& w, const uint4* xs, int c, int,
                                             const half2&, int& acc) {
    const uint4 xv = xs[c];
    acc = __dp4a(int(w.x), int(xv.x), acc);
    acc = __dp4a(int(w.y), int(xv.y), acc);
    acc = __dp4a(int(w.z), int(xv.z), acc);
    acc = __dp4a(int(w.w), int(xv.w), acc);
  }
};

template <>
struct ChunkDot<kW4> {
  using Acc = float;
  // xs is "planar": plane j (j = word index 0..3 within a chunk) holds the 8
  // activations of word j of every chunk, so lanes read consecutive 16 bytes.
  __device__ __forceinline__ static void run(const uint4& w, const uint4* xs, int c, int nch,
                                             const half2& s2, float& acc) {
    const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
    const half2 k1032 = __float2half2_rn(1032.0f);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint4 xv = xs[j * nch + c];
      const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
      half2 hacc = __float2half2_rn(0.0f);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const half2 q = __hsub2(u2h2(lop3_and_or(wv[j] >> (4 * i), 0x000F000Fu, 0x64006400u)), k1032);
        const half2 wd = __hmul2(q, s2);  // = fp16((q-8)*s), the W4 dequant contract
        hacc = __hfma2(wd, u2h2(xw[i]), hacc);
      }
      const float2 f = __half22float2(hacc);
      acc += f.x + f.y;
    }
  }
};

// Activation prologue into shared memory, for NT token rows of x (fp32 [NT, k]).
// Token t's activations live at smem + t * k * elt (planar layout for W4).
template <int FMT, int PRO, int NT>
__device__ __forceinline__ void prologue(const float* __restrict__ x, const half* __restrict__ gamma,
                                         float eps, int k, int T, uint8_t* smem, float* red,
                                         float* xscale) {
  for (int t = 0; t < NT; ++t) {
    if (t >= T) {  // padding token: zero activations
      const int bytes = FMT == kINT8 ? k : 2 * k;
      for (int i = threadIdx.x; i < bytes / 16; i += kThreads)
        reinterpret_cast<uint4*>(smem + size_t(t) * bytes)[i] = make_uint4(0, 0, 0, 0);
      if (threadIdx.x == 0) xscale[t] = 0.0f;
      continue;
    }
    const float* xt = x + size_t(t) * k;
    float r = 1.0f;
    if (PRO == kProNorm) {
      float ss = 0.0f;
      for (int i = threadIdx.x; i < k; i += kThreads) ss = fmaf(xt[i], xt[i], ss);
      ss = block_sum(ss, red);
      r = 1.0f / sqrtf(ss / float(k) + eps);
    }
    auto act = [&](int i) -> float {
      return PRO == kProNorm ? (xt[i] * r) * __half2float(gamma[i]) : xt[i];
    };
    if (FMT == kINT8) {
      float amax = 0.0f;
      for (int i = threadIdx.x; i < k; i += kThreads) amax = fmaxf(amax, fabsf(act(i)));
      amax = block_max(amax, red);
      const float s = amax / 127.0f;
      int8_t* xq = reinterpret_cast<int8_t*>(smem) + size_t(t) * k;
      for (int i = threadIdx.x; i < k; i += kThreads) {
        const float v = amax > 0.0f ? rintf(act(i) / s) : 0.0f;
        xq[i] = static_cast<int8_t>(fminf(fmaxf(v, -127.0f), 127.0f));
      }
      if (threadIdx.x == 0) xscale[t] = s;
    } else if (FMT == kFP16) {
      half* xh = reinterpret_cast<half*>(smem) + size_t(t) * k;
      for (int i = threadIdx.x; i < k; i += kThreads) xh[i] = __float2half_rn(act(i));
    } else {
      half* xh = reinterpret_cast<half*>(smem) + size_t(t) * k;
      const int nch = k / 32;
      for (int i = threadIdx.x; i < k; i += kThreads) {
        const int c = i >> 5, j = (i >> 3) & 3, o = i & 7;
        xh[(j * nch + c) * 8 + o] = __float2half_rn(act(i));
      }
    }
    __syncthreads();
  }
  __syncthreads();
}

template <int FMT, int PRO, int EPI, int NT>
__global__ void __launch_bounds__(kThreads) gemv_kernel(const uint8_t* __restrict__ w,
                                                        const void* __restrict__ ws, int n, int k,
                                                        const float* __restrict__ x, int T,
                                                        const half* __restrict__ gamma, float eps,
                                                        float* __restrict__ y) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ float red[32];
  __shared__ float xscale[NT];
  using Dot = ChunkDot<FMT>;
  using Acc = typename Dot::Acc;
  constexpr int E = Fmt<FMT>::kElemsPerChunk;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nch = k / E;  // 16-byte chunks per row
  const size_t row_bytes = size_t(nch) * 16;
  const int tok_stride16 = (FMT == kINT8 ? k : 2 * k) / 16;  // uint4s per token in smem
  const int npairs = n >> 1;
  const int groups = (nch + 32 * kUnroll - 1) / (32 * kUnroll);
  const int pair_stride = gridDim.x * kWarps;
  int pair = blockIdx.x * kWarps + warp;

  // Issue the first weight chunks before the prologue.
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
  if (pair < npairs) load(pair, 0, buf);

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
          half2 s0 = __float2half2_rn(0.f), s1 = s0;
          if (FMT == kW4) {
            const half* sc = static_cast<const half*>(ws);
            const int groups_k = k / kW4Group;
            s0 = __half2half2(sc[size_t(2 * pair) * groups_k + (c >> 2)]);
            s1 = __half2half2(sc[size_t(2 * pair + 1) * groups_k + (c >> 2)]);
          }
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            Dot::run(buf[0][u], xs + t * tok_stride16, c, nch, s0, acc0[t]);
            Dot::run(buf[1][u], xs + t * tok_stride16, c, nch, s1, acc1[t]);
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
      if (lane == 0 && t < T) {
        if (EPI == kEpiStore) {
          y[size_t(t) * n + 2 * pair] = v0;
          y[size_t(t) * n + 2 * pair + 1] = v1;
        } else if (EPI == kEpiResid) {
          y[size_t(t) * n + 2 * pair] += v0;
          y[size_t(t) * n + 2 * pair + 1] += v1;
        } else {
          y[size_t(t) * (n / 2) + pair] = silu(v0) * v1;
        }
      }
    }
  }
}

template <int FMT, int PRO, int EPI, int NT>
void launch_t(const LinearW& W, const float* x, int T, const half* gamma, float eps, float* y,
              cudaStream_t st) {
  const int npairs = W.n / 2;
  const int grid = std::max(1, std::min(ceil_div(npairs, kWarps), kNumSMs * 16));
  const size_t smem = size_t(NT) * (FMT == kINT8 ? size_t(W.k) : size_t(W.k) * 2);
  static bool attr_done = false;  // per template instance
  if (!attr_done) {
    MSW_CUDA(cudaFuncSetAttribute(gemv_kernel<FMT, PRO, EPI, NT>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr_done = true;
  }
  gemv_kernel<FMT, PRO, EPI, NT><<<grid, kThreads, smem, st>>>(
      static_cast<const uint8_t*>(W.w), W.s, W.n, W.k, x, T, gamma, eps, y);
  MSW_LAUNCH_CHECK();
}

template <int FMT, int NT>
void dispatch_nt(const LinearW& W, int pro, int epi, const float* x, int T, const half* gamma,
                 float eps, float* y, cudaStream_t st) {
#define MSW_GEMV_CASE(P, E) \
  if (pro == P && epi == E) return launch_t<FMT, P, E, NT>(W, x, T, gamma, eps, y, st);
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
  if (T <= kGemvMaxTokens) return dispatch_nt<FMT, kGemvMaxTokens>(W, pro, epi, x, T, gamma, eps, y, st);
  throw ConfigErr("gemv: too many tokens");
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

}  // namespace

void launch_gemv(const LinearW& W, int pro, int epi, const float* x, int T, const half* gamma,
                 float eps, float* y, cudaStream_t st) {
  if (W.n % 2 != 0 || W.k % 128 != 0) throw ConfigErr("gemv: n must be even, k a multiple of 128");
  if (T < 1 || T > kGemvMaxTokens) throw ConfigErr("gemv: 1..6 tokens");
  switch (W.fmt) {
    case kFP16: return dispatch_fmt<kFP16>(W, pro, epi, x, T, gamma, eps, y, st);
    case kINT8: return dispatch_fmt<kINT8>(W, pro, epi, x, T, gamma, eps, y, st);
    case kW4: return dispatch_fmt<kW4>(W, pro, epi, x, T, gamma, eps, y, st);
    default: throw ConfigErr("gemv: bad weight format");
  }
}

void launch_gemv_i8_acc(const int8_t* w, const int8_t* x, int n, int k, int* acc, cudaStream_t st) {
  if (k % 16 != 0) throw ConfigErr("gemv_i8_acc: k must be a multiple of 16");
  gemv_i8_acc_kernel<<<ceil_div(n, kWarps), kThreads, 0, st>>>(w, x, n, k, acc);
  MSW_LAUNCH_CHECK();
}

}  // namespace msw
