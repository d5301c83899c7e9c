// Shared device helpers for the sm_100a mode executor.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <stdexcept>
#include <string>

namespace msw {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ConfigErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DataErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define MSW_CUDA(expr)                                                            \
  do {                                                                            \
    cudaError_t e_ = (expr);                                                      \
    if (e_ != cudaSuccess)                                                        \
      throw ::msw::CudaError(std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define MSW_LAUNCH_CHECK() MSW_CUDA(cudaGetLastError())

constexpr int kNumSMs = 148;
constexpr int kKvBlock = 16;
constexpr int kW4Group = 128;

// ---- K16 deterministic init --------------
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t tensor_key(uint64_t seed, uint64_t tid) {
  return mix64(seed ^ (tid * 0xD1B54A32D192ED03ull));
}
// uniform in [-1, 1), 2^-23 resolution, exact in fp32
__host__ __device__ __forceinline__ float unif(uint64_t key, uint64_t idx) {
  const uint64_t r = mix64(key + idx);
  const int32_t u = static_cast<int32_t>(r >> 40);
  return static_cast<float>(u - 8388608) * 1.1920928955078125e-07f;
}

constexpr uint64_t kTidDraftBase = 1ull << 32;
constexpr uint64_t kTidEmbed = 1;
constexpr uint64_t kTidFinalNorm = 3;
__host__ __device__ constexpr uint64_t tid_layer(int l, int kind) {
  return 256ull + 16ull * static_cast<uint64_t>(l) + static_cast<uint64_t>(kind);
}
enum TensorKind { kQ = 0, kK, kV, kO, kGate, kUp, kDown, kAttnNorm, kFfnNorm };
constexpr uint64_t kSuccSalt = 0x5375636365737373ull;
constexpr uint64_t kAgreeSalt = 0x4167726565416772ull;

// ---- small device utilities -----------------------------------------------
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Streaming 128-bit weight load: read-only path, no L1 allocation.
__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ float silu(float g) { return g / (1.0f + expf(-g)); }
// Prefill-GEMM epilogue SiLU: ex2.approx-based exp and the fast divide (a
// few ulp of fp32 from silu(); the product is rounded to fp16 or int8 before
// the next linear). silu() cost ~40 instructions per element, which made the
// gate_up GEMM's epilogue ~1/3 of its time at 128 x 256 tiles.
__device__ __forceinline__ float silu_fast(float g) { return __fdividef(g, 1.0f + __expf(-g)); }

// Intra-CTA timeline probes, compiled only into the diagnostics build
// (-DMSW_TRACE -> libmsw_engine_trace.so, scripts/gemv_timeline.py). Slot i of
// CTA b receives clock64() relative to the CTA's first probe; slot 15 holds
// %globaltimer at probe 0 (cross-CTA skew). Zero cost in the product build.
#ifdef MSW_TRACE
__device__ __forceinline__ unsigned long long* msw_trace_buf();
#define MSW_TP(i)                                                                  \
  do {                                                                             \
    unsigned long long* tb_ = msw_trace_buf();                                     \
    if (tb_) {                                                                     \
      unsigned long long c_ = clock64();                                           \
      if ((i) == 0) {                                                              \
        unsigned long long g_;                                                     \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_));                     \
        tb_[blockIdx.x * 16 + 15] = g_;                                            \
        tb_[blockIdx.x * 16 + 14] = c_;                                            \
      }                                                                            \
      tb_[blockIdx.x * 16 + (i)] = c_;                                             \
    }                                                                              \
  } while (0)
#else
#define MSW_TP(i) \
  do {            \
  } while (0)
#endif

// Programmatic dependent launch: everything before pdl_wait() may only touch
// data the previous kernel does not write (weights); pdl_trigger() lets the
// next kernel in the stream start its own weight prefetch early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }

// ---- mbarrier / bulk-async-copy helpers (shared by the TMA-fed kernels)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "MSW_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra MSW_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Orders this thread's prior generic-proxy shared-memory accesses (and those
// it acquired) before its subsequent async-proxy operations (bulk copies).
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// 1-D bulk async copy global -> shared, completion counted on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Same, with an L2 cache policy (createpolicy): weights streamed once per step
// use evict_first so the KV cache and activations stay L2-resident.
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes,
                                              uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
      "%2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// Named barrier over `threads` threads (id 1..15; 0 is __syncthreads).
// The NON-aligned form: every thread arrives individually, so a warp that
// reaches it diverged (the compiler does not know an inline-asm barrier needs
// reconvergence) is still counted correctly. `bar.sync` is
// barrier.sync.aligned, which is undefined for a diverged warp: compute-
// sanitizer synccheck flagged it at the GEMV prologue barriers, and it let
// consumer warps start on partially written activations (the sporadic stale
// tiles of the FP16 6-token K=14336 GEMV, scripts/repro_gemv_t6.py).
__device__ __forceinline__ void named_sync(int id, int threads) {
  asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// Bulk L2 prefetch of a contiguous byte range (TMA unit, no registers used).
// Address and size must be multiples of 16.
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// Prefetch [p, p+bytes) in <= 64 KB pieces, spread over the calling warp's lanes.
__device__ __forceinline__ void prefetch_l2_range(const void* p, size_t bytes, int lane) {
  const char* c = static_cast<const char*>(p);
  constexpr size_t kPiece = 64 * 1024;
  const size_t pieces = (bytes + kPiece - 1) / kPiece;
  for (size_t i = lane; i < pieces; i += 32) {
    const size_t off = i * kPiece;
    const size_t n = bytes - off < kPiece ? bytes - off : kPiece;
    prefetch_l2(c + off, static_cast<uint32_t>(n & ~size_t(15)));
  }
}

// A/B experiment switches (MSW_NO_PDL, MSW_L2NEXT_KB, MSW_GEMV_W4_GENERIC,
// MSW_SKIP) are read only by the diagnostics build (-DMSW_TRACE); the product
// library ignores the environment.
inline const char* diag_env(const char* name) {
#ifdef MSW_TRACE
  return std::getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

// Launch with the programmatic-stream-serialization attribute (PDL).
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  static const bool pdl_off = diag_env("MSW_NO_PDL") != nullptr;  // A/B experiments
  cfg.attrs = attr;
  cfg.numAttrs = pdl_off ? 0 : 1;
  MSW_CUDA(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
}

// Block-wide reductions for <= 1024 threads; `red` needs 32 floats of smem.
__device__ __forceinline__ float block_sum(float v, float* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  float t = lane < nw ? red[lane] : 0.0f;
  return warp_sum(t);
}
__device__ __forceinline__ float block_max(float v, float* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  float t = lane < nw ? red[lane] : -3.402823466e38f;
  return warp_max(t);
}

inline int ceil_div(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

}  // namespace msw
