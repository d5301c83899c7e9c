// T > 1 token linears (prefill, speculative verify, continuous-batching steps).
//
// prep_act: per-token RMSNorm + activation handling (fp16 rounding or per-token
// int8 quantisation), identical to the GEMV prologue contract.
// gemm_tiled: portable CUDA-core tile kernel, used for shapes the tcgen05
// kernel (gemm_tc.cu) does not take and as its correctness fallback-free
// reference on device; W8A8 accumulates in int32 exactly.
#include "kernels.cuh"

namespace msw {
namespace {

// One CTA per token; the row is read from HBM once into registers (float4,
// up to kPrepV per thread) and normalised, reduced and converted there: one
// read pass instead of two (FP16) or three (INT8: sum of squares, absmax,
// quantise) over the row.
constexpr int kPrepThreads = 512;
constexpr int kPrepV = 8;  // float4 per thread: K <= 16384

__global__ void __launch_bounds__(kPrepThreads)
    prep_act_kernel(int fmt, const float* __restrict__ x, int K, const half* __restrict__ gamma,
                    float eps, half* __restrict__ xh, int8_t* __restrict__ xq,
                    float* __restrict__ xscale) {
  __shared__ float red[32];
  // PDL: the row comes from the previous kernel, and xh / xq may still be
  // read by the GEMM before that; the next GEMM may launch (and stream its
  // weights) as soon as every row CTA is past this point
  pdl_wait();
  pdl_trigger();
  const size_t t = blockIdx.x;
  const int n4 = K / 4;
  const float4* xr = reinterpret_cast<const float4*>(x + t * K);
  float4 v[kPrepV];
#pragma unroll
  for (int j = 0; j < kPrepV; ++j) {
    const int i = threadIdx.x + j * kPrepThreads;
    v[j] = i < n4 ? xr[i] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (gamma != nullptr) {
    float ss = 0.0f;
#pragma unroll
    for (int j = 0; j < kPrepV; ++j)
      ss = fmaf(v[j].x, v[j].x, fmaf(v[j].y, v[j].y, fmaf(v[j].z, v[j].z, fmaf(v[j].w, v[j].w, ss))));
    ss = block_sum(ss, red);
    const float r = 1.0f / sqrtf(ss / float(K) + eps);
#pragma unroll
    for (int j = 0; j < kPrepV; ++j) {
      const int i = threadIdx.x + j * kPrepThreads;
      if (i < n4) {
        const half2* g = reinterpret_cast<const half2*>(gamma) + 2 * i;
        const float2 g0 = __half22float2(g[0]), g1 = __half22float2(g[1]);
        v[j].x = (v[j].x * r) * g0.x;
        v[j].y = (v[j].y * r) * g0.y;
        v[j].z = (v[j].z * r) * g1.x;
        v[j].w = (v[j].w * r) * g1.y;
      }
    }
  }
  if (fmt == kINT8) {
    float amax = 0.0f;
#pragma unroll
    for (int j = 0; j < kPrepV; ++j)
      amax = fmaxf(amax, fmaxf(fmaxf(fabsf(v[j].x), fabsf(v[j].y)), fmaxf(fabsf(v[j].z), fabsf(v[j].w))));
    amax = block_max(amax, red);
    const float s = amax / 127.0f;
    auto q = [&](float u) -> int8_t {
      const float w = amax > 0.0f ? rintf(u / s) : 0.0f;
      return static_cast<int8_t>(fminf(fmaxf(w, -127.0f), 127.0f));
    };
#pragma unroll
    for (int j = 0; j < kPrepV; ++j) {
      const int i = threadIdx.x + j * kPrepThreads;
      if (i < n4)
        reinterpret_cast<char4*>(xq + t * K)[i] = make_char4(q(v[j].x), q(v[j].y), q(v[j].z), q(v[j].w));
    }
    if (threadIdx.x == 0) xscale[t] = s;
  } else {
#pragma unroll
    for (int j = 0; j < kPrepV; ++j) {
      const int i = threadIdx.x + j * kPrepThreads;
      if (i < n4) {
        half2* o = reinterpret_cast<half2*>(xh + t * K) + 2 * i;
        o[0] = __floats2half2_rn(v[j].x, v[j].y);
        o[1] = __floats2half2_rn(v[j].z, v[j].w);
      }
    }
  }
}

constexpr int BM = 64;  // tokens per tile
constexpr int BN = 64;  // weight rows per tile
constexpr int BK = 32;

template <int FMT>
__device__ __forceinline__ float dequant(const uint8_t* w, const void* ws, const uint8_t* wz, int n,
                                         int k, int K) {
  if (FMT == kFP16) {
    return __half2float(reinterpret_cast<const half*>(w)[size_t(n) * K + k]);
  } else {
    const uint32_t word = reinterpret_cast<const uint32_t*>(w)[size_t(n) * (K / 8) + k / 8];
    const int idx = k & 7;
    const int pos = (idx >> 1) + 4 * (idx & 1);
    const int zero = wz ? int(wz[size_t(n) * (K / kW4Group) + k / kW4Group]) : 8;  // AWQ / GPTQ
    const int q = int((word >> (4 * pos)) & 0xF) - zero;
    const half s = static_cast<const half*>(ws)[size_t(n) * (K / kW4Group) + k / kW4Group];
    return __half2float(__hmul(__int2half_rn(q), s));
  }
}

template <int FMT, int EPI>
__global__ void __launch_bounds__(256)
    gemm_tiled_kernel(const uint8_t* __restrict__ w, const void* __restrict__ ws, int N, int K,
                      const half* __restrict__ xh, const int8_t* __restrict__ xq,
                      const float* __restrict__ xscale, int T, float* __restrict__ y,
                      const uint8_t* __restrict__ wz) {
  using Acc = typename std::conditional<FMT == kINT8, int, float>::type;
  __shared__ Acc Xs[BK][BM + 4];
  __shared__ Acc Ws[BK][BN + 4];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16 threads, 4x4 each
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  Acc acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0;

  for (int k0 = 0; k0 < K; k0 += BK) {
    for (int e = threadIdx.x; e < BK * BM; e += 256) {
      const int kk = e % BK, mm = e / BK;
      const int m = m0 + mm, k = k0 + kk;
      Acc v = 0;
      if (m < T) {
        if (FMT == kINT8) v = Acc(xq[size_t(m) * K + k]);
        else v = Acc(__half2float(xh[size_t(m) * K + k]));
      }
      Xs[kk][mm] = v;
    }
    for (int e = threadIdx.x; e < BK * BN; e += 256) {
      const int kk = e % BK, nn = e / BK;
      const int n = n0 + nn, k = k0 + kk;
      Acc v = 0;
      if (n < N) {
        if (FMT == kINT8) v = Acc(reinterpret_cast<const int8_t*>(w)[size_t(n) * K + k]);
        else v = Acc(dequant<FMT>(w, ws, wz, n, k, K));
      }
      Ws[kk][nn] = v;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < BK; ++kk) {
      Acc a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = Xs[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Ws[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += a[i] * b[j];
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= T) continue;
    float v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (EPI == kEpiRaw) {
        v[j] = __int_as_float(int(acc[i][j]));
      } else if (FMT == kINT8) {
        v[j] = n < N ? (float(acc[i][j]) * xscale[m]) * static_cast<const float*>(ws)[n] : 0.0f;
      } else {
        v[j] = float(acc[i][j]);
      }
    }
#pragma unroll
    for (int j = 0; j < 4; j += 2) {
      const int n = n0 + tx * 4 + j;
      if (n >= N) continue;
      if (EPI == kEpiStore || EPI == kEpiRaw) {
        y[size_t(m) * N + n] = v[j];
        y[size_t(m) * N + n + 1] = v[j + 1];
      } else if (EPI == kEpiResid) {
        y[size_t(m) * N + n] += v[j];
        y[size_t(m) * N + n + 1] += v[j + 1];
      } else {
        y[size_t(m) * (N / 2) + n / 2] = silu(v[j]) * v[j + 1];
      }
    }
  }
}

template <int FMT>
void gemm_fmt(const LinearW& W, int epi, const half* xh, const int8_t* xq, const float* xscale,
              int T, float* y, cudaStream_t st) {
  const dim3 grid(ceil_div(W.n, BN), ceil_div(T, BM));
  const uint8_t* w = static_cast<const uint8_t*>(W.w);
  if (epi == kEpiStore)
    gemm_tiled_kernel<FMT, kEpiStore><<<grid, 256, 0, st>>>(w, W.s, W.n, W.k, xh, xq, xscale, T, y, W.z);
  else if (epi == kEpiResid)
    gemm_tiled_kernel<FMT, kEpiResid><<<grid, 256, 0, st>>>(w, W.s, W.n, W.k, xh, xq, xscale, T, y, W.z);
  else if (epi == kEpiSwiglu)
    gemm_tiled_kernel<FMT, kEpiSwiglu><<<grid, 256, 0, st>>>(w, W.s, W.n, W.k, xh, xq, xscale, T, y, W.z);
  else if (FMT == kINT8 && epi == kEpiRaw)
    gemm_tiled_kernel<FMT, kEpiRaw><<<grid, 256, 0, st>>>(w, W.s, W.n, W.k, xh, xq, xscale, T, y, W.z);
  else
    throw ConfigErr("gemm: bad epilogue");
  MSW_LAUNCH_CHECK();
}

}  // namespace

void launch_prep_act(int fmt, const float* x, int T, int K, const half* gamma, float eps, half* xh,
                     int8_t* xq, float* xscale, cudaStream_t st) {
  if (K % 4 || K > kPrepThreads * kPrepV * 4) throw ConfigErr("prep_act: K must be a multiple of 4, <= 16384");
  launch_pdl(prep_act_kernel, dim3(T), dim3(kPrepThreads), 0, st, fmt, x, K, gamma, eps, xh, xq, xscale);
}

void launch_gemm(const LinearW& W, int epi, const half* xh, const int8_t* xq, const float* xscale,
                 int T, float* y, cudaStream_t st) {
  if (gemm_tc_supported(W)) return launch_gemm_tc(W, epi, xh, xq, xscale, T, y, st);
  if (W.k % BK != 0 || W.n % 2 != 0) throw ConfigErr("gemm: bad shape");
  switch (W.fmt) {
    case kFP16: return gemm_fmt<kFP16>(W, epi, xh, xq, xscale, T, y, st);
    case kINT8: return gemm_fmt<kINT8>(W, epi, xh, xq, xscale, T, y, st);
    case kW4: return gemm_fmt<kW4>(W, epi, xh, xq, xscale, T, y, st);
    default: throw ConfigErr("gemm: bad format");
  }
}

}  // namespace msw
