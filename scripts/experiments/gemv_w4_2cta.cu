// EXPERIMENT, NOT BUILT (measured negative).
// A two-CTA-per-SM batch-1 W4 decode GEMV (<= 108 KB smem, 320 threads) with
// dynamic tile claiming, meant to let the next linear's CTA stream its ring
// while the current one drains. It compiled against an L2Next with
// rounds/w_round/s_round fields and a gemv.cu dispatch hook; both were
// removed with it. In the 8B W4 decode step it measured 593 tok/s (all four
// linears) and 652 (qkv/o only) against 682 for the one-CTA kernel: eight
// consumer warps sustain only ~30 weights/cycle/SM (LOP3 half-rate ALU pipe,
// x fragments from shared memory = 2/3 of the LDS wavefronts), static ranges
// let two CTAs of one linear share an SM, and a cross-CTA tile combine cost
// ~2.3 us per launch.
// Batch-1 W4 (GPTQ uint4b8, group 128) decode GEMV, sized for TWO CTAs per SM.
//
// Why two: a decode step is a chain of GEMVs, each an HBM stream of 8-60 MB
// (1.3-9 us at the HBM rate). With one 190 KB CTA per SM, kernel N+1's CTA
// cannot become resident on an SM until kernel N's CTA there has exited, so
// every GEMV paid its ring fill (~1.3 us to the first consumed stage) and its
// drain on the critical path: back to back, o (8.7 MB) took 3.9 us and qkv
// (13 MB) 5.0 us. Here a CTA uses <= 104 KB of shared memory and 320 threads
// (<= 102 registers), so the CTA of the NEXT linear is resident while this one
// drains: its producer warp streams its first stages before
// griddepcontrol.wait (the weights do not depend on the previous kernel), and
// HBM never idles between linears.
//
// Layout and arithmetic are those of the tile-fragment W4 path (gemv.cu):
// 16-row tiles of 512-byte chunks (16 rows x 64 k = four k16 MMA steps; even
// steps dequantise as 1024 + q against x, odd steps as 1024 + 16q against
// x/16, one lop3 per fp16 pair); the per-group offset 1032*Sx_even +
// 72*Sx_odd is removed in fp32 before the per-row group scale.
//
// Roles: 8 consumer warps (each takes 4 chunks = two 128-k groups of every
// 16 KB stage), 1 producer warp (cp.async.bulk ring), 1 epilogue warp.
// Activations: ONE fp16 copy, with the odd-step positions pre-scaled by 1/16
// and laid out so that a lane's B fragments for a step pair are one LDS.128.
//
// The prologue reads x ONCE (registers) after griddepcontrol.wait: it is the
// only dependent global access on the critical path between two linears.
// The inner loop keeps four independent MMA accumulator chains (even / odd
// k16 steps of two groups) so 8 warps hide the mma.sync latency.
#include "kernels.cuh"
#include "mma_frag.cuh"

namespace msw {
namespace {

constexpr int kC = 8;                     // consumer warps
constexpr int kThr = (kC + 2) * 32;       // + producer + epilogue
constexpr int kCThr = kC * 32;
constexpr int kS = 32;                    // chunks per stage
constexpr int kChunk = 512;
constexpr int kStageB = kS * kChunk;      // 16 KB
constexpr int kCPW = kS / kC;             // 4 chunks per warp per stage
constexpr int kMaxStg = 6;
constexpr int kTS = 3;                    // per-tile scale slots
constexpr int kSmemCap = 108 * 1024;      // dynamic; 2 x (108 + static + 1 reserved) <= 228 KB

#ifdef MSW_TRACE
// back-to-back timeline (diagnostics build only): per (launch, CTA) 8 words
// [smid, start, consumers past PDL wait, first stage consumed, consumers done,
//  epilogue done, -, -] in globaltimer ns; launch index = CTA ticket / grid.
__device__ unsigned long long* g_w4c_trace = nullptr;
__device__ unsigned g_w4c_seq = 0;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long g;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
  return g;
}
#define W4C_TP(slot_)                                                      \
  do {                                                                     \
    if (trace_row) trace_row[slot_] = gtimer();                            \
  } while (0)
#else
#define W4C_TP(slot_) \
  do {                \
  } while (0)
#endif

// Tile claim counters: launch j uses counter j & 1 (the next linear's CTAs
// may claim while this one's are still claiming); the last claim of a launch
// (value ntiles + grid - 1) resets its counter to 0. Module globals, so no
// allocation can fall inside a stream capture.
__device__ unsigned g_w4c_claim[2];

// half index of x[k] (k even; pairs stay adjacent). Per 32-k block (k16 steps
// 2m, 2m+1), lane tq owns 16 bytes: [x(2tq), x(2tq+1), x(2tq+8), x(2tq+9) of
// the even step | the same four of the odd step, times 1/16].
__device__ __forceinline__ int xslot(int k) {
  const int u = k & 31, s = u >> 4, v = u & 15;
  return (k & ~31) + ((v & 7) >> 1) * 8 + s * 4 + (v >> 3) * 2 + (v & 1);
}

template <int EPI>
__device__ __forceinline__ void store_rows(float* y, int n, int row, float v0, float v1) {
  if (EPI == kEpiStore) {
    y[row] = v0;
    y[row + 1] = v1;
  } else if (EPI == kEpiResid) {
    y[row] += v0;
    y[row + 1] += v1;
  } else {
    y[row / 2] = silu(v0) * v1;  // rows (2i, 2i+1) = (gate_i, up_i)
  }
  (void)n;
}

// x fp32 [k] -> (RMSNorm) -> fp16 in the xslot layout + per-group offsets,
// k = 1024 XV. Thread t holds float4 i = t + 256 j (j < XV) in registers
// between the sum of squares and the conversion: warp w covers k in
// [128 (w + 8 j), +128) = one scale group per j, and lane bit 2 is the
// k16-step parity.
template <int PRO, int XV>
__device__ __forceinline__ void prologue(const float* __restrict__ x, const half* __restrict__ gamma,
                                         float eps, half* xh, float* corr, float* red) {
  constexpr int k = XV * 1024;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float4* xt = reinterpret_cast<const float4*>(x);
  float4 v[XV];
#pragma unroll
  for (int j = 0; j < XV; ++j) v[j] = xt[tid + j * kCThr];
  float r = 1.0f;
  if (PRO == kProNorm) {
    float ss = 0.0f;
#pragma unroll
    for (int j = 0; j < XV; ++j)
      ss = fmaf(v[j].x, v[j].x, fmaf(v[j].y, v[j].y, fmaf(v[j].z, v[j].z, fmaf(v[j].w, v[j].w, ss))));
    ss = warp_sum(ss);
    if (lane == 0) red[warp] = ss;
    named_sync(1, kCThr);
    float t = lane < kC ? red[lane] : 0.0f;
    t = warp_sum(t);
    r = 1.0f / sqrtf(t / float(k) + eps);
  }
  const half2 sixteenth = __float2half2_rn(0.0625f);
#pragma unroll
  for (int j = 0; j < XV; ++j) {
    const int i = tid + j * kCThr;
    float4 a = v[j];
    if (PRO == kProNorm) {
      const half2* gm = reinterpret_cast<const half2*>(gamma) + 2 * i;
      const float2 g0 = __half22float2(gm[0]), g1 = __half22float2(gm[1]);
      a.x = (a.x * r) * g0.x;
      a.y = (a.y * r) * g0.y;
      a.z = (a.z * r) * g1.x;
      a.w = (a.w * r) * g1.y;
    }
    half2 lo = __floats2half2_rn(a.x, a.y), hi = __floats2half2_rn(a.z, a.w);
    const float2 lf = __half22float2(lo), hf = __half22float2(hi);
    const int kk = 4 * i;
    if (kk & 16) {  // odd k16 step: stored as x/16 (exact power-of-two scaling)
      lo = __hmul2(lo, sixteenth);
      hi = __hmul2(hi, sixteenth);
    }
    *reinterpret_cast<half2*>(xh + xslot(kk)) = lo;
    *reinterpret_cast<half2*>(xh + xslot(kk + 2)) = hi;
    float gs = (lf.x + lf.y) + (hf.x + hf.y);
    gs += __shfl_xor_sync(0xffffffffu, gs, 1);
    gs += __shfl_xor_sync(0xffffffffu, gs, 2);
    gs += __shfl_xor_sync(0xffffffffu, gs, 8);
    gs += __shfl_xor_sync(0xffffffffu, gs, 16);
    const float odd = __shfl_sync(0xffffffffu, gs, 4);
    if (lane == 0) corr[i / 32] = 1032.0f * gs + 72.0f * odd;
  }
  named_sync(1, kCThr);
}

// mma.sync without `volatile`, so independent accumulator chains interleave
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int PRO, int EPI, int XV>
__global__ void __launch_bounds__(kThr, 2)
    gemv_w4c_kernel(const uint8_t* __restrict__ wtf, const half* __restrict__ ws, int n,
                    const float* __restrict__ x, const half* __restrict__ gamma, float eps,
                    float* __restrict__ y, int n_stages, int parity, const L2Next nx) {
  unsigned* const claim = &g_w4c_claim[parity];
  constexpr int k = XV * 1024;
  constexpr int chunks_tile = k / 64;
  constexpr int spt = chunks_tile / kS;  // stages per tile
  constexpr int groups_k = k / kW4Group;
  constexpr int tile_sbytes = 16 * groups_k * 2;  // one tile's scales: 16 consecutive rows
  static_assert(chunks_tile % kS == 0, "a tile is a whole number of stages");
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full[kMaxStg], empty[kMaxStg];
  __shared__ uint64_t sfull[kTS], sfree[kTS];  // per-tile scale slots
  __shared__ uint64_t tile_full[2], tile_free[2];
  __shared__ int slot_tile[kTS];                // claimed tile of a scale slot, -1 = done
  __shared__ int part_tile[2];
  __shared__ float red[kC];
  __shared__ __align__(16) float part[2][kC][16];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = n / 16;
  half* xh = reinterpret_cast<half*>(smem);
  float* corr = reinterpret_cast<float*>(smem + size_t(2) * k);
  uint8_t* sc_smem = smem + ((size_t(2) * k + size_t(groups_k) * 4 + 127) & ~size_t(127));
  uint8_t* ring = sc_smem + kTS * tile_sbytes;

#ifdef MSW_TRACE
  __shared__ unsigned long long* trace_sh;
  if (threadIdx.x == 0) {
    trace_sh = nullptr;
    if (g_w4c_trace) {
      const unsigned t = atomicAdd(&g_w4c_seq, 1u);
      const unsigned launch = t / gridDim.x;
      if (launch < 512) {
        trace_sh = g_w4c_trace + (size_t(launch) * kNumSMs + blockIdx.x) * 8;
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        trace_sh[0] = smid;
        trace_sh[1] = gtimer();
      }
    }
  }
#endif
  if (threadIdx.x == 0) {
    for (int s = 0; s < n_stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kC);
    }
    for (int s = 0; s < kTS; ++s) {
      mbar_init(&sfull[s], 1);
      mbar_init(&sfree[s], kC);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tile_full[b], kCThr);  // every consumer lane arrives
      mbar_init(&tile_free[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
#ifdef MSW_TRACE
  unsigned long long* const trace_row = (threadIdx.x == 0 || threadIdx.x == kCThr + 32) ? trace_sh : nullptr;
#endif

  if (warp == kC) {  // producer: claims tiles and streams them, ahead of the PDL wait
    if (lane == 0) {
      unsigned next = atomicAdd(claim, 1u);  // first claim before anything else
      int s = 0, ts = 0;
      uint32_t phase = 0, tphase = 0;
      for (;;) {
        const unsigned t = next;
        if (t < unsigned(ntiles)) next = atomicAdd(claim, 1u);  // one claim in flight
        mbar_wait(&sfree[ts], tphase ^ 1);
        if (t >= unsigned(ntiles)) {  // this CTA is done; the last claim of the launch resets
          slot_tile[ts] = -1;
          mbar_arrive(&sfull[ts]);
          if (t == unsigned(ntiles) + gridDim.x - 1) *claim = 0u;
          break;
        }
        slot_tile[ts] = int(t);
        mbar_expect_tx(&sfull[ts], tile_sbytes);
        bulk_g2s(sc_smem + ts * tile_sbytes, reinterpret_cast<const uint8_t*>(ws) + size_t(t) * tile_sbytes,
                 tile_sbytes, &sfull[ts]);
        const uint8_t* src = wtf + size_t(t) * chunks_tile * kChunk;
#pragma unroll 1
        for (int j = 0; j < spt; ++j) {
          mbar_wait(&empty[s], phase ^ 1);
          mbar_expect_tx(&full[s], kStageB);
          bulk_g2s(ring + size_t(s) * kStageB, src + size_t(j) * kStageB, kStageB, &full[s]);
          if (++s == n_stages) {
            s = 0;
            phase ^= 1;
          }
        }
        if (++ts == kTS) {
          ts = 0;
          tphase ^= 1;
        }
      }
      l2_next_prefetch(nx);
    }
    pdl_wait();
    pdl_trigger();
    return;
  }
  if (warp == kC + 1) {  // epilogue: 8 per-warp partials -> y
    pdl_wait();
    pdl_trigger();
    const int rp = lane >> 2, q = lane & 3;  // row pair, warp pair
    for (int i = 0;; ++i) {
      const int b = i & 1;
      mbar_wait(&tile_full[b], (i >> 1) & 1);
      const int tile = part_tile[b];
      const float* p1 = &part[b][0][0];
      float v0 = p1[(2 * q) * 16 + 2 * rp] + p1[(2 * q + 1) * 16 + 2 * rp];
      float v1 = p1[(2 * q) * 16 + 2 * rp + 1] + p1[(2 * q + 1) * 16 + 2 * rp + 1];
      v0 += __shfl_xor_sync(0xffffffffu, v0, 1);
      v1 += __shfl_xor_sync(0xffffffffu, v1, 1);
      v0 += __shfl_xor_sync(0xffffffffu, v0, 2);
      v1 += __shfl_xor_sync(0xffffffffu, v1, 2);
      __syncwarp();
      if (lane == 0) mbar_arrive(&tile_free[b]);  // partials are in registers
      if (tile < 0) break;
      if (q == 0) store_rows<EPI>(y, n, tile * 16 + 2 * rp, v0, v1);
    }
    W4C_TP(5);
    return;
  }

  // consumers
  pdl_wait();
  W4C_TP(2);
  pdl_trigger();
  prologue<PRO, XV>(x, gamma, eps, xh, corr, red);
  const int g = lane >> 2, tq = lane & 3;
  const uint8_t* xl = reinterpret_cast<const uint8_t*>(xh) + tq * 16;
  int slot = 0, ts = 0;
  uint32_t phase = 0, tphase = 0;
#pragma unroll 1
  for (int i = 0;; ++i) {
    mbar_wait(&sfull[ts], tphase);
    const int tile = slot_tile[ts];
    const int b = i & 1;
    if (i >= 2) mbar_wait(&tile_free[b], ((i >> 1) - 1) & 1);
    if (tile < 0) {  // no more tiles: hand the epilogue its stop marker
      if (threadIdx.x == 0) part_tile[b] = -1;
      mbar_arrive(&tile_full[b]);
      break;
    }
    if (i == 0) W4C_TP(3);
    const half* sc_h = reinterpret_cast<const half*>(sc_smem + ts * tile_sbytes);
    float acc0 = 0.f, acc2 = 0.f;
#pragma unroll 1
    for (int j2 = 0; j2 < spt; ++j2) {
      mbar_wait(&full[slot], phase);
      const uint4* stage = reinterpret_cast<const uint4*>(ring + size_t(slot) * kStageB) + warp * kCPW * 32 + lane;
      uint4 a4[kCPW];
#pragma unroll
      for (int j = 0; j < kCPW; ++j) a4[j] = stage[j * 32];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);  // operands are in registers
      if (++slot == n_stages) {
        slot = 0;
        phase ^= 1;
      }
      const int c0 = j2 * kS + warp * kCPW;  // this warp's first chunk within the tile
      // two groups (chunk pairs), each with separate even- and odd-step
      // accumulators: four independent mma chains of four
      float ce[2][4] = {}, co[2][4] = {};
#pragma unroll
      for (int j = 0; j < kCPW; ++j) {
        const uint32_t wv[4] = {a4[j].x, a4[j].y, a4[j].z, a4[j].w};
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          const uint4 xb = *reinterpret_cast<const uint4*>(xl + ((c0 + j) * 2 + p) * 64);
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
          mma16816(ce[j >> 1], a_lo, xb.x, xb.y);
          mma16816(co[j >> 1], a_hi, xb.z, xb.w);
        }
      }
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        const int grp = (c0 >> 1) + jj;
        const float slo = __half2float(sc_h[g * groups_k + grp]);
        const float shi = __half2float(sc_h[(g + 8) * groups_k + grp]);
        const float kk = corr[grp];
        acc0 = fmaf(slo, (ce[jj][0] + co[jj][0]) - kk, acc0);
        acc2 = fmaf(shi, (ce[jj][2] + co[jj][2]) - kk, acc2);
      }
    }
    if (tq == 0) {  // column 0 (the one token): rows g and g + 8
      part[b][warp][g] = acc0;
      part[b][warp][g + 8] = acc2;
    }
    if (threadIdx.x == 0) part_tile[b] = tile;
    __syncwarp();
    if (lane == 0) mbar_arrive(&sfree[ts]);     // this warp is done with the tile's scales
    mbar_arrive(&tile_full[b]);                  // per-lane release of its own stores
    if (++ts == kTS) {
      ts = 0;
      tphase ^= 1;
    }
  }
  W4C_TP(4);
}

struct Plan {
  int grid, stages;
  size_t smem;
};

Plan plan(int n, int k) {
  Plan p{};
  p.grid = std::max(1, std::min(n / 16, kNumSMs));
  const int groups = k / kW4Group;
  const size_t fixed = ((size_t(2) * k + size_t(groups) * 4 + 127) & ~size_t(127)) +
                       size_t(kTS) * 16 * groups * 2;
  p.stages = fixed >= size_t(kSmemCap) ? 0 : std::min<int>(kMaxStg, int((kSmemCap - fixed) / kStageB));
  p.smem = fixed + size_t(p.stages) * kStageB;
  return p;
}

thread_local unsigned t_launch_seq = 0;

template <int PRO, int EPI, int XV>
void launch_t(const LinearW& W, const float* x, const half* gamma, float eps, float* y,
              const L2Next& nx, cudaStream_t st) {
  const Plan p = plan(W.n, W.k);
  if (p.stages < 3) throw ConfigErr("gemv(w4c): shared memory budget exceeded");
  static bool attr_done = false;
  if (!attr_done) {
    MSW_CUDA(cudaFuncSetAttribute(gemv_w4c_kernel<PRO, EPI, XV>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemCap));
    MSW_CUDA(cudaFuncSetAttribute(gemv_w4c_kernel<PRO, EPI, XV>,
                                  cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    attr_done = true;
  }
  const int parity = int(t_launch_seq++ & 1u);
  launch_pdl(gemv_w4c_kernel<PRO, EPI, XV>, dim3(p.grid), dim3(kThr), p.smem, st,
             static_cast<const uint8_t*>(W.w_tf), static_cast<const half*>(W.s), W.n, x, gamma,
             eps, y, p.stages, parity, nx);
}

template <int PRO, int EPI>
void launch_k(const LinearW& W, const float* x, const half* gamma, float eps, float* y,
              const L2Next& nx, cudaStream_t st) {
  if (W.k == 4096) return launch_t<PRO, EPI, 4>(W, x, gamma, eps, y, nx, st);
  if (W.k == 14336) return launch_t<PRO, EPI, 14>(W, x, gamma, eps, y, nx, st);
  throw ConfigErr("gemv(w4c): k must be 4096 or 14336");
}

}  // namespace

#ifdef MSW_TRACE
extern "C" int msw_w4c_trace_set(void* buf) {
  const unsigned zero = 0;
  if (cudaMemcpyToSymbol(g_w4c_seq, &zero, sizeof(zero)) != cudaSuccess) return 1;
  return cudaMemcpyToSymbol(g_w4c_trace, &buf, sizeof(buf)) == cudaSuccess ? 0 : 1;
}
#endif

bool gemv_w4c_supported(const LinearW& W) {
  // the Llama-3.1-8B decode shapes (x is held in registers by the prologue)
#if defined(MSW_W4C_OFF)  // A/B build switches (scripts/build_variant.sh)
  return false && W.n;
#elif defined(MSW_W4C_ALL)
  return W.fmt == kW4 && W.w_tf && W.n % 16 == 0 && (W.k == 4096 || W.k == 14336) &&
         plan(W.n, W.k).stages >= 3;
#else
  return W.fmt == kW4 && W.w_tf && W.n % 16 == 0 && W.k == 4096 && W.n <= 8192 &&
         plan(W.n, W.k).stages >= 3;
#endif
}

void launch_gemv_w4c(const LinearW& W, int pro, int epi, const float* x, const half* gamma,
                     float eps, float* y, const L2Next& nx, cudaStream_t st) {
#define MSW_W4C_CASE(P, E) \
  if (pro == P && epi == E) return launch_k<P, E>(W, x, gamma, eps, y, nx, st);
  MSW_W4C_CASE(kProPlain, kEpiStore)
  MSW_W4C_CASE(kProPlain, kEpiResid)
  MSW_W4C_CASE(kProPlain, kEpiSwiglu)
  MSW_W4C_CASE(kProNorm, kEpiStore)
  MSW_W4C_CASE(kProNorm, kEpiResid)
  MSW_W4C_CASE(kProNorm, kEpiSwiglu)
#undef MSW_W4C_CASE
  throw ConfigErr("gemv(w4c): bad prologue/epilogue");
}

}  // namespace msw
