// Blackwell tensor-core linear for T > kGemvMaxTokens tokens (prefill,
// continuous-batching steps): tcgen05.mma with the accumulator in TMEM.
//
// Swap-AB: the WEIGHT tile is the MMA's M=128 operand (128 output features,
// K-major, exactly the row-major [n, k] storage) and the activation tile is the
// N operand (BN tokens, K-major [t, k]); D[n, t] accumulates in TMEM (lane =
// feature, column = token). This keeps M at 128 for any token count, so small
// continuous-batching steps (T = 16..64) still run full-width UMMAs.
//
// Per CTA (one 128 x BN output tile, or one K-slice of it):
//   warp 0 (one lane) : TMA producer, 4-stage smem ring (SWIZZLE_128B tiles)
//   warp 1 (one lane) : MMA issuer (tcgen05.mma, commit -> empty barrier)
//   warp 2            : TMEM allocation owner
//   warp 3 (one lane, W4) : TMA producer of the packed weights, 8-stage ring
//   warps 0-3         : epilogue, tcgen05.ld 32x32b, fused store / residual
//                       add / SwiGLU / W8A8 rescale
//   warps 4-7 (W4)    : dequantisers: packed uint4b8 (smem) + fp16 group
//                       scale -> fp16 (q-8)*s written in the SW128 K-major
//                       layout the UMMA descriptor reads (no int4 UMMA on sm_100a)
// kind::f16 for FP16 and W4, kind::i8 (int32 accumulate, exact) for W8A8.
//
// Small token counts leave most SMs idle with one CTA per 128-row tile (a
// continuous-batching step or a 128-token prefill of a 4096-row projection is
// 32 tiles), so K is split over up to 8 CTAs that form a thread-block cluster
// and reduce their partial tiles through distributed shared memory, in a
// fixed order (deterministic; exact int32 for W8A8).
#include <cuda.h>

#include <mutex>
#include <type_traits>
#include <unordered_map>

#include "kernels.cuh"

namespace msw {
namespace {

constexpr int kMaxStages = 8;  // operand ring depth cap (barrier arrays)
constexpr int kTileM = 128;     // weight rows per CTA (UMMA M)
constexpr int kTileKBytes = 128;  // one SW128 row per k-tile

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B canonical layout
// (8-row x 128-byte atoms, SBO = 1024 B between atoms along M/N, LBO = 16 B).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = uint64_t((saddr & 0x3FFFF) >> 4);
  d |= uint64_t(1) << 16;           // LBO (16 B; unused for swizzled K-major)
  d |= uint64_t(1024 >> 4) << 32;   // SBO
  d |= uint64_t(1) << 46;           // descriptor version (sm_100)
  d |= uint64_t(2) << 61;           // SWIZZLE_128B
  return d;
}

template <int FMT, int BN, int M = kTileM>
__device__ __forceinline__ constexpr uint32_t instr_desc() {
  // c_format bits 4-5 (F32=1, S32=2); a/b format bits 7-9 / 10-12 (F16=0; INT8 signed=1);
  // K-major A and B; N>>3 at bits 17-22; M>>4 at bits 24-28.
  return (FMT == kINT8 ? (2u << 4) | (1u << 7) | (1u << 10) : (1u << 4)) |
         (uint32_t(BN >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

template <int FMT>
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                     uint32_t accumulate) {
  if (FMT == kINT8) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
  }
}
// A operand from TMEM (the W4 dequantisers' fp16 tile), B from shared memory
__device__ __forceinline__ void umma_ts(uint32_t tmem_d, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem_d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
// CTA-pair MMA (cta_group::2, issued by the pair's leader): D[256 x N] with A
// rows 0..127 from the leader's shared memory and 128..255 from the peer's (same
// offsets), B columns split between the two CTAs, D rows in each CTA's TMEM.
template <int FMT>
__device__ __forceinline__ void umma_pair(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
  if (FMT == kINT8) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
  }
}
// arrive on the barrier at this offset in both CTAs of the pair once the MMAs complete
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(uint16_t(3))
      : "memory");
}
// TMA into this CTA's shared memory, completion counted on the pair leader's
// mbarrier at the same offset (peer bit of the shared::cluster address cleared)
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint64_t* bar,
                                                 int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// Split-K CTAs of one output tile form a thread-block cluster along z; the
// partial tiles are reduced through distributed shared memory (below).
constexpr int kMaxSplit = 8;  // portable cluster size
constexpr int kPkStages = 8;  // W4: packed-weight ring depth (4 KB stages)

// CG = 2: CTA pair (cta_group::2) over two adjacent weight-row tiles sharing
// a token tile; each CTA holds its 128 weight rows and HALF of the token
// tile, so one k-tile moves 16 + 16 KB through a CTA's shared memory instead
// of 16 + 32 KB. With 128 x 256 tiles the single-CTA ring (TMA writes + MMA
// reads ~190 B/clk/SM at the f16 rate) is shared-memory-bandwidth bound.
template <int FMT, int BN, int CG = 1>
struct TcCfg {
  static constexpr bool kIsW4 = FMT == kW4;
  static constexpr int kElt = FMT == kINT8 ? 1 : 2;
  static constexpr int kTileK = kTileKBytes / kElt;           // elements per k-tile
  static constexpr int kUmmaK = FMT == kINT8 ? 32 : 16;       // elements per UMMA
  static constexpr int kABytes = kTileM * kTileKBytes;        // 16 KB
  static constexpr int kBBytes = (BN / CG) * kTileKBytes;  // this CTA's token rows
  static constexpr int kPkBytes = kIsW4 ? kTileM * 32 : 0;    // 128 rows x 8 packed words
  // W4: 8 dequantiser warps (two per weight row, 4 packed words each) keep the
  // fp16 operand production ahead of the MMA (4 warps bounded W4 prefill below FP16)
  static constexpr int kDqWarps = 8;
  static constexpr int kThreads = kIsW4 ? 128 + kDqWarps * 32 : 128;
  // W4 with 128 x 256 tiles: the dequantised A tile goes to TMEM (tcgen05.st,
  // MMA with A from TMEM) instead of a swizzled shared-memory tile: the
  // operand path then moves 36 KB of shared memory per k-tile (B + packed
  // words) instead of 68 KB (B + packed + A written and read), which bounded
  // the W4 prefill GEMM below FP16. TMEM: accumulator [0, 256), A stages of
  // 32 columns (128 rows x 64 k fp16) from column 256.
  static constexpr bool kAT = kIsW4 && BN == 256;
  static constexpr int kARing = kAT ? 0 : kABytes;  // A bytes per shared-memory stage
  static constexpr uint32_t kColA = BN;
  static constexpr int kTmemCols = kAT ? 512 : (BN < 32 ? 32 : BN);
  // operand ring as deep as ~220 KB of shared memory allows (one CTA per SM):
  // a short prefill / CB step streams weights at HBM rate only with enough
  // bytes in flight per SM (latency x bandwidth / 148)
  static constexpr int kStageBytes = kARing + kBBytes;
  // W4 with 128 x 256 tiles: a 4-deep packed ring (16 KB) leaves room for a
  // 4th operand stage (the dequantisers can only fill a slot the MMA freed)
  static constexpr int kPk = kIsW4 && BN > 128 ? 4 : kPkStages;
  static constexpr int kStagesFit = (220 * 1024 - kPk * kPkBytes) / kStageBytes;
  static constexpr int kStages = kStagesFit < kMaxStages ? kStagesFit : kMaxStages;
  static constexpr int kRingBytes = kStages * (kARing + kBBytes) + kPk * kPkBytes;
  static_assert(!kAT || int(kColA) + kStages * 32 <= kTmemCols, "A stages must fit TMEM");
  static constexpr int kSmem = kRingBytes + 1024 /*align*/ + 512 /*barriers*/;
  // split-K partial tile [BN][128] (fp32 / int32), staged in the A ring once
  // every MMA has completed; up to ks-1 incoming column slices ((ks-1)/ks of
  // a tile) land in the B ring
  static_assert(kStages >= (BN > 128 ? 3 : 4), "ring too shallow");
  // split-K (BN <= 128 only; long prefills fill the machine without it)
  static constexpr bool kCanSplit = BN <= 128 && CG == 1;
  static_assert(CG == 1 || (!kIsW4 && BN == 256), "CTA pairs: FP16 / INT8 with 128 x 256 tiles");
  static_assert(!kCanSplit || BN * kTileM * 4 <= kStages * kABytes, "partial tile must fit the A ring");
  static_assert(!kCanSplit || BN * kTileM * 4 <= kStages * kBBytes, "incoming slices must fit the B ring");
};

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// Bulk copy of `bytes` from this CTA's smem to the same-named buffers of
// cluster CTA `rank`: dst / bar are local addresses mapped into the peer.
__device__ __forceinline__ void bulk_s2s_peer(void* dst, const void* src, uint32_t bytes,
                                              uint64_t* bar, uint32_t rank) {
  uint32_t rdst, rbar;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rdst) : "r"(smem_u32(dst)), "r"(rank));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          rdst),
      "r"(smem_u32(src)), "r"(bytes), "r"(rbar)
      : "memory");
}

template <int FMT, int BN, int EPI, int CG>
__global__ void __launch_bounds__(TcCfg<FMT, BN, CG>::kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   int N, int K, int T, const void* __restrict__ wscale,
                   const float* __restrict__ xscale, float* __restrict__ y, int ksplit,
                   const uint8_t* __restrict__ wzero) {
  using C = TcCfg<FMT, BN, CG>;
  using Acc32 = typename std::conditional<FMT == kINT8, int, float>::type;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::kStages * C::kARing;
  uint8_t* sP = sB + C::kStages * C::kBBytes;  // W4 packed ring
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kRingBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* pfull = empty + C::kStages;
  uint64_t* pempty = pfull + C::kPk;
  uint64_t* done = pempty + C::kPk;
  uint64_t* rbar = done + 1;  // split-K: incoming partial slices
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rbar + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // grid x = token tiles, y = weight-row tiles: the CTAs that share one
  // 128-row weight slab are adjacent in launch order, so a long prefill
  // (T = 1024: 8 token tiles) reads each weight byte from HBM once and from
  // L2 for the other tiles (weight-tile-major order read it 8 times: 1.89 GB
  // of DRAM for a 235 MB FP16 gate_up)
  // CTA pairs sit along x (the pair is two x-adjacent CTAs of a (2,1,1)
  // cluster): x = 2 * token tile + rank, y = weight-row tile pair
  const int t0 = (CG == 2 ? (blockIdx.x >> 1) : blockIdx.x) * BN;
  const int n0 = (CG == 2 ? blockIdx.y * 2 + (blockIdx.x & 1) : blockIdx.y) * kTileM;
  // split-K: blockIdx.z (= cluster rank) owns k-tiles [kb0, kb0 + nk)
  const int nk_all = K / C::kTileK;
  const int nk_per = (nk_all + ksplit - 1) / ksplit;
  const int kb0 = blockIdx.z * nk_per;
  const int nk = max(0, min(nk_all - kb0, nk_per));

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], C::kIsW4 ? 1 + C::kDqWarps : 1);  // TMA arrive (+ dequant warps)
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < C::kPk; ++s) {
      mbar_init(&pfull[s], 1);
      mbar_init(&pempty[s], C::kDqWarps);
    }
    mbar_init(done, 1);
    mbar_init(rbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
  }
  if (warp == 2) {
    if constexpr (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(C::kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(C::kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t prank = CG == 2 ? cluster_ctarank() : 0;  // 0: the pair's leader
  if (CG == 2) cluster_sync_all();  // both CTAs' barriers initialised before any pair traffic

  if (warp == 0 && lane == 0) {
    // ---- TMA producer: activation tiles (+ weight tiles for FP16 / INT8).
    // PDL: the first ring's weight tiles are requested before
    // griddepcontrol.wait (weights are never written by a kernel), the
    // activation tiles only after it
    const int npre = C::kIsW4 ? 0 : min(nk, C::kStages);
    if constexpr (CG == 2) {
      // pair: the leader arms its full barrier for both CTAs' bytes; both
      // CTAs' loads complete on it. A: this CTA's 128 weight rows; B: its
      // half of the token tile.
      constexpr uint32_t kPairBytes = 2u * (C::kABytes + C::kBBytes);
      const int tb = t0 + int(prank) * (BN / 2);
      for (int kb = 0; kb < npre; ++kb) {  // fresh slots: no empty wait
        if (prank == 0) mbar_expect_tx(&full[kb], kPairBytes);
        tma_load_2d_pair(sA + kb * C::kABytes, &tmA, &full[kb], (kb0 + kb) * C::kTileK, n0);
      }
      pdl_wait();
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % C::kStages;
        const uint32_t ph = (kb / C::kStages) & 1;
        if (kb >= npre) {
          mbar_wait(&empty[s], ph ^ 1);
          if (prank == 0) mbar_expect_tx(&full[s], kPairBytes);
          tma_load_2d_pair(sA + s * C::kABytes, &tmA, &full[s], (kb0 + kb) * C::kTileK, n0);
        }
        tma_load_2d_pair(sB + s * C::kBBytes, &tmB, &full[s], (kb0 + kb) * C::kTileK, tb);
      }
      // drain: every slot released by the leader's MMAs, so no pair commit
      // arrives on this CTA's barriers after it exits
      for (int kb = nk; kb < nk + C::kStages; ++kb)
        if (kb >= C::kStages) mbar_wait(&empty[kb % C::kStages], ((kb / C::kStages) & 1) ^ 1);
    } else {
      for (int kb = 0; kb < npre; ++kb) {  // fresh slots: no empty wait
        mbar_expect_tx(&full[kb], C::kABytes + C::kBBytes);
        tma_load_2d(sA + kb * C::kABytes, &tmA, &full[kb], (kb0 + kb) * C::kTileK, n0);
      }
      pdl_wait();
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % C::kStages;
        const uint32_t ph = (kb / C::kStages) & 1;
        if (kb >= npre) {
          mbar_wait(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], C::kIsW4 ? C::kBBytes : C::kABytes + C::kBBytes);
          if (!C::kIsW4) tma_load_2d(sA + s * C::kABytes, &tmA, &full[s], (kb0 + kb) * C::kTileK, n0);
        }
        tma_load_2d(sB + s * C::kBBytes, &tmB, &full[s], (kb0 + kb) * C::kTileK, t0);
      }
    }
  } else if (warp == 1 && lane == 0 && CG == 2) {
    // ---- pair MMA issuer (leader only): M = 256 over both CTAs' weight rows
    if (prank == 0) {
      constexpr uint32_t idesc = instr_desc<FMT, BN, 2 * kTileM>();
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % C::kStages;
        const uint32_t ph = (kb / C::kStages) & 1;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t a0 = smem_u32(sA + s * C::kABytes);
        const uint32_t b0 = smem_u32(sB + s * C::kBBytes);
#pragma unroll
        for (int k = 0; k < C::kTileK / C::kUmmaK; ++k) {
          const uint32_t off = k * C::kUmmaK * C::kElt;
          umma_pair<FMT>(tmem, sw128_desc(a0 + off), sw128_desc(b0 + off), idesc, (kb | k) != 0);
        }
        umma_commit_pair(&empty[s]);
      }
      umma_commit_pair(done);
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer
    constexpr uint32_t idesc = instr_desc<FMT, BN>();
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % C::kStages;
      const uint32_t ph = (kb / C::kStages) & 1;
      mbar_wait(&full[s], ph);
      tc_fence_after();
      const uint32_t a0 = smem_u32(sA + s * C::kARing);
      const uint32_t b0 = smem_u32(sB + s * C::kBBytes);
#pragma unroll
      for (int k = 0; k < C::kTileK / C::kUmmaK; ++k) {
        const uint32_t off = k * C::kUmmaK * C::kElt;  // bytes along the swizzled row
        if constexpr (C::kAT)  // 16 k = 8 TMEM columns of fp16 pairs per MMA
          umma_ts(tmem, tmem + C::kColA + uint32_t(s) * 32 + uint32_t(k) * 8, sw128_desc(b0 + off),
                  idesc, (kb | k) != 0);
        else
          umma<FMT>(tmem, sw128_desc(a0 + off), sw128_desc(b0 + off), idesc, (kb | k) != 0);
      }
      umma_commit(&empty[s]);
    }
    umma_commit(done);  // with nk == 0 this still arrives (no MMA issued: D stays unwritten)
  } else if (C::kIsW4 && warp == 3 && lane == 0) {
    // ---- W4 packed-weight producer: 128 rows x 64 k (8 words per row, 4 KB)
    // per k-tile, C::kPk deep, ahead of the dequantisers
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % C::kPk;
      const uint32_t ph = (kb / C::kPk) & 1;
      mbar_wait(&pempty[s], ph ^ 1);
      fence_proxy_async();  // dequantisers' generic reads of this slot before the TMA overwrite
      mbar_expect_tx(&pfull[s], C::kPkBytes);
      tma_load_2d(sP + s * C::kPkBytes, &tmA, &pfull[s], (kb0 + kb) * 8, n0);
    }
  } else if (C::kIsW4 && warp >= 4) {
    // ---- W4 dequantisers: thread (r, hf) owns packed words 4hf..4hf+3 (k
    // 32hf..32hf+31) of weight row n0 + r of every k-tile: packed words from
    // the smem ring -> fp16 (q-8)*s in the SW128 K-major layout the UMMA
    // descriptor reads (no int4 UMMA on sm_100a)
    const int r = (threadIdx.x - 128) & 127, hf = (threadIdx.x - 128) >> 7;
    const half* srow = static_cast<const half*>(wscale) + size_t(n0 + r) * (K / kW4Group);
    // (1024 + q) - (1024 + zero): zero 8 (GPTQ uint4b8) or the AWQ zero point of the group
    const uint8_t* zrow = wzero ? wzero + size_t(n0 + r) * (K / kW4Group) : nullptr;
    const half2 k1032 = __float2half2_rn(1032.0f);
    for (int kb = 0; kb < nk; ++kb) {
      const int ps = kb % C::kPk;
      const uint32_t pph = (kb / C::kPk) & 1;
      const int s = kb % C::kStages;
      const uint32_t ph = (kb / C::kStages) & 1;
      const int grp = ((kb0 + kb) * 64) / kW4Group;
      const half2 s2 = __half2half2(srow[grp]);
      const half2 kz = zrow ? __float2half2_rn(1024.0f + float(zrow[grp])) : k1032;
      mbar_wait(&pfull[ps], pph);
      const uint4 p0 = reinterpret_cast<const uint4*>(sP + ps * C::kPkBytes + r * 32)[hf];
      __syncwarp();
      if (lane == 0) mbar_arrive(&pempty[ps]);
      mbar_wait(&empty[s], ph ^ 1);
      const uint32_t words[4] = {p0.x, p0.y, p0.z, p0.w};
      if constexpr (C::kAT) {
        // TMEM lane = row r (this warp's lane quarter is (warp & 3) = r / 32),
        // columns 16 hf .. 16 hf + 15 of stage s = k pairs 32 hf .. 32 hf + 31
        tc_fence_after();  // the MMAs that read this stage (empty barrier) before the overwrite
        uint32_t out[16];
#pragma unroll
        for (int cc = 0; cc < 4; ++cc)
#pragma unroll
          for (int i = 0; i < 4; ++i) {  // nibbles i, i+4 of word cc = elements 8cc+2i, +1
            uint32_t u = lop3_and_or(words[cc] >> (4 * i), 0x000F000Fu, 0x64006400u);
            const half2 q = __hsub2(*reinterpret_cast<const half2*>(&u), kz);
            const half2 wv = __hmul2(q, s2);
            out[4 * cc + i] = *reinterpret_cast<const uint32_t*>(&wv);
          }
        tmem_st16(tmem + (uint32_t((warp & 3) * 32) << 16) + C::kColA + uint32_t(s) * 32 + 16 * hf, out);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
      } else {
        uint8_t* rowp = sA + s * C::kABytes + r * 128;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {  // chunk c = k 8c..8c+7 = packed word c
          const int c = 4 * hf + cc;
          uint32_t out[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            uint32_t u = lop3_and_or(words[cc] >> (4 * i), 0x000F000Fu, 0x64006400u);
            const half2 q = __hsub2(*reinterpret_cast<const half2*>(&u), kz);
            const half2 wv = __hmul2(q, s2);
            out[i] = *reinterpret_cast<const uint32_t*>(&wv);
          }
          *reinterpret_cast<uint4*>(rowp + ((c ^ (r & 7)) << 4)) = make_uint4(out[0], out[1], out[2], out[3]);
        }
        fence_async_smem();  // generic-proxy stores -> visible to the tensor core
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[s]);
    }
  }

  // the next kernel may launch once every CTA's mainloop is issued (it
  // waits for this grid's completion before reading y)
  pdl_trigger();
  // ---- epilogue (warps 0-3): TMEM lane = weight row, column = token
  __syncwarp();  // reconverge the producer / MMA lanes before .sync.aligned TMEM loads
  const int row = (warp & 3) * 32 + lane;
  const int n = n0 + row;
  float ws = 1.0f;
  if (FMT == kINT8 && warp < 4) ws = static_cast<const float*>(wscale)[n];
  // column j of this tile (token t0 + j), raw accumulator bits u
  // residual epilogue: the 16 y values of a column batch are read together
  // (independent loads in flight) instead of one read-modify-write round trip
  // per column; emit() of a batch uses them
  float prev[16];
  auto emit = [&](int j, uint32_t u) {
    const int t = t0 + j;
    if (EPI == kEpiRaw) {  // INT8 test entry: the int32 accumulator itself
      if (t < T) reinterpret_cast<uint32_t*>(y)[size_t(t) * N + n] = u;
      return;
    }
    const float v = FMT == kINT8 ? (float(int(u)) * (t < T ? xscale[t] : 0.0f)) * ws
                                 : __uint_as_float(u);
    if (EPI == kEpiSwiglu) {  // rows (2i, 2i+1) = (gate_i, up_i) sit in adjacent lanes
      const float up = __shfl_xor_sync(0xffffffffu, v, 1);
      if (t < T && (lane & 1) == 0) y[size_t(t) * (N / 2) + (n >> 1)] = silu_fast(v) * up;
    } else if (t < T) {
      if (EPI == kEpiStore) y[size_t(t) * N + n] = v;
      else y[size_t(t) * N + n] = prev[j & 15] + v;  // prev: this 16-column batch's y
    }
  };
  if (warp < 4) {
    // residual epilogue: pull this row's y values for the tile's tokens into L2
    // while the mainloop runs, so the epilogue's reads are L2 hits
    if (EPI == kEpiResid) {  // split-K: only the columns this cluster rank finishes
      const int c0 = ksplit == 1 ? 0 : int(cluster_ctarank()) * (BN / ksplit);
      const int c1 = min(ksplit == 1 ? BN : c0 + BN / ksplit, T - t0);
      for (int j = c0; j < c1; ++j)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(y + size_t(t0 + j) * N + n));
    }
    mbar_wait(done, 0);
    tc_fence_after();
  }
  const uint32_t trow = tmem + (uint32_t((warp & 3) * 32) << 16);
  if (ksplit == 1) {
    if (warp < 4) {
#pragma unroll 1
      for (int j0 = 0; j0 < BN; j0 += 16) {
        uint32_t r[16];
        tmem_ld16(trow + j0, r);
#pragma unroll
        for (int j = 0; j < 16; ++j) {  // residual: all 16 reads in flight before the adds
          if (EPI == kEpiResid) prev[j] = t0 + j0 + j < T ? y[size_t(t0 + j0 + j) * N + n] : 0.0f;
        }
        if (EPI == kEpiSwiglu) {
          // column pairs: the even lane (gate) finishes column j, the odd lane
          // (up) column j + 1, one shuffle each way: one SiLU per lane per two
          // columns instead of 16 idle odd lanes per column
#pragma unroll
          for (int j = 0; j < 16; j += 2) {
            const int ta = t0 + j0 + j, tb = ta + 1;
            const float v0 = FMT == kINT8 ? (float(int(r[j])) * (ta < T ? xscale[ta] : 0.0f)) * ws
                                          : __uint_as_float(r[j]);
            const float v1 = FMT == kINT8 ? (float(int(r[j + 1])) * (tb < T ? xscale[tb] : 0.0f)) * ws
                                          : __uint_as_float(r[j + 1]);
            const bool odd = lane & 1;
            const float got = __shfl_xor_sync(0xffffffffu, odd ? v0 : v1, 1);
            const float g = odd ? got : v0, u = odd ? v1 : got;
            const int t = odd ? tb : ta;
            if (t < T) y[size_t(t) * (N / 2) + (n >> 1)] = silu_fast(g) * u;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) emit(j0 + j, r[j]);
        }
      }
    }
  } else if constexpr (C::kCanSplit) {
    // Deterministic split-K through distributed shared memory: every CTA of
    // the cluster stages its raw partial tile [BN][128] in its own (now idle)
    // A ring; after a cluster barrier each CTA pushes column slice r of its
    // partial to CTA r with one bulk copy (cp.async.bulk smem -> peer smem,
    // completion on the receiver's mbarrier), and CTA r sums its slice over
    // the ks partials in rank order and runs the epilogue for it. INT8
    // partials are int32, so the result is the exact int32 sum, scaled once.
    // No global workspace, no atomics, no tail CTA.
    uint32_t* red = reinterpret_cast<uint32_t*>(sA);
    uint32_t* recv = reinterpret_cast<uint32_t*>(sB);  // idle B ring: (ks-1) incoming slices
    const int cpr = BN / ksplit;  // columns owned per rank (>= 2)
    const uint32_t slice_bytes = uint32_t(cpr) * kTileM * 4;
    const int rank = int(cluster_ctarank());
    if (threadIdx.x == 0) mbar_expect_tx(rbar, uint32_t(ksplit - 1) * slice_bytes);
    if (warp < 4) {
#pragma unroll 1
      for (int j0 = 0; j0 < BN; j0 += 16) {
        uint32_t r[16];
        tmem_ld16(trow + j0, r);
#pragma unroll
        for (int j = 0; j < 16; ++j) red[(j0 + j) * kTileM + row] = nk > 0 ? r[j] : 0u;
      }
    }
    fence_async_smem();  // generic stores -> visible to the bulk-copy (async) proxy
    cluster_sync_all();  // partials staged, every CTA's mainloop done, receivers armed
    if (threadIdx.x == 0) {
      for (int r = 0; r < ksplit; ++r) {
        if (r == rank) continue;
        const int idx = rank < r ? rank : rank - 1;  // this CTA's slot among r's senders
        bulk_s2s_peer(recv + size_t(idx) * cpr * kTileM, red + size_t(r) * cpr * kTileM,
                      slice_bytes, rbar, uint32_t(r));
      }
    }
    if (warp < 4) {
      mbar_wait(rbar, 0);
#pragma unroll 1
      for (int c = 0; c < cpr; ++c) {
        Acc32 a = 0;
        for (int z = 0; z < ksplit; ++z) {
          const uint32_t u = z == rank ? red[(rank * cpr + c) * kTileM + row]
                                       : recv[((z < rank ? z : z - 1) * cpr + c) * kTileM + row];
          if (FMT == kINT8) a += Acc32(int(u));
          else a += Acc32(__uint_as_float(u));
        }
        if (EPI == kEpiResid) {
          const int tt = t0 + rank * cpr + c;
          prev[(rank * cpr + c) & 15] = tt < T ? y[size_t(tt) * N + n] : 0.0f;
        }
        emit(rank * cpr + c, FMT == kINT8 ? uint32_t(int(a)) : __float_as_uint(float(a)));
      }
    }
    cluster_sync_all();  // peers have read this CTA's partials before it exits
  }
  tc_fence_before();
  __syncthreads();
  if (CG == 2) cluster_sync_all();  // the pair's MMAs and commits are complete in both CTAs
  if (warp == 2) {
    if constexpr (CG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "r"(C::kTmemCols));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "r"(C::kTmemCols));
  }
}

// ---- host side: tensor maps through the driver entry point (no -lcuda)
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    fn = reinterpret_cast<EncodeFn>(p);
  });
  if (!fn) throw CudaError("cuTensorMapEncodeTiled unavailable");
  return fn;
}

// 2-D K-major tile map: rows x k elements, box = box_rows x box_bytes.
CUtensorMap make_map(const void* base, CUtensorMapDataType dt, int elt_bytes, uint64_t rows,
                     uint64_t k, int box_rows, int box_bytes, CUtensorMapSwizzle swz) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {k, rows};
  const cuuint64_t strides[1] = {k * elt_bytes};
  const cuuint32_t box[2] = {cuuint32_t(box_bytes / elt_bytes), cuuint32_t(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
  return m;
}
CUtensorMap make_sw128_map(const void* base, int elt_bytes, uint64_t rows, uint64_t k, int box_rows) {
  return make_map(base, elt_bytes == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                  elt_bytes, rows, k, box_rows, kTileKBytes, CU_TENSOR_MAP_SWIZZLE_128B);
}

// Split-K factor: only when the output tiles fill less than half of the
// resident CTA slots (a continuous-batching step, a short prefill of a
// 4096-row projection), split K over the largest power of two (<= 8, each
// split keeping >= 8 k-tiles) that keeps the CTAs within one wave. Fuller
// grids run unsplit: short-lived split CTAs cost more in pipeline fill and
// reduction than the wave tail they save.
int choose_split(int tiles, int nk, int slots) {
  int ks = 1;
  while (ks < kMaxSplit && tiles * ks * 2 <= slots && nk / (ks * 2) >= 8) ks *= 2;
  return ks;
}

template <int FMT, int BN, int EPI, int CG>
void launch_bn(const LinearW& W, const void* xact, const float* xscale, int T, float* y,
               cudaStream_t st) {
  using C = TcCfg<FMT, BN, CG>;
  static int per_sm = 0;
  if (!per_sm) {
    MSW_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<FMT, BN, EPI, CG>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
    MSW_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gemm_tc_kernel<FMT, BN, EPI, CG>,
                                                           C::kThreads, C::kSmem));
    per_sm = std::max(per_sm, 1);
  }
  const int elt = C::kElt;
  // FP16 / INT8: weight tiles 128 rows x 128 B, SWIZZLE_128B; W4: packed
  // words 128 rows x 8 words (32 B), unswizzled (the dequantisers swizzle)
  const CUtensorMap ta =
      FMT == kW4 ? make_map(W.w, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, W.n, W.k / 8, kTileM, 32,
                            CU_TENSOR_MAP_SWIZZLE_NONE)
                 : make_sw128_map(W.w, elt, W.n, W.k, kTileM);
  const CUtensorMap tb = make_sw128_map(xact, elt, T, W.k, BN / CG);
  const int tiles = (W.n / kTileM) * ((T + BN - 1) / BN);
  const int ksplit = C::kCanSplit ? choose_split(tiles, W.k / C::kTileK, kNumSMs * per_sm) : 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = CG == 2 ? dim3(2 * ((T + BN - 1) / BN), W.n / kTileM / 2, 1)
                        : dim3((T + BN - 1) / BN, W.n / kTileM, ksplit);
  cfg.blockDim = dim3(C::kThreads);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = ksplit;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (weights before the wait)
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  MSW_CUDA(cudaLaunchKernelEx(&cfg, gemm_tc_kernel<FMT, BN, EPI, CG>, ta, tb, W.n, W.k, T, W.s, xscale,
                              y, ksplit, FMT == kW4 ? W.z : static_cast<const uint8_t*>(nullptr)));
}

template <int FMT, int EPI>
void launch_fmt_epi(const LinearW& W, const void* x, const float* xs, int T, float* y,
                    cudaStream_t st) {
  if (T <= 16) return launch_bn<FMT, 16, EPI, 1>(W, x, xs, T, y, st);
  if (T <= 32) return launch_bn<FMT, 32, EPI, 1>(W, x, xs, T, y, st);
  if (T <= 64) return launch_bn<FMT, 64, EPI, 1>(W, x, xs, T, y, st);
  if (T <= 128) return launch_bn<FMT, 128, EPI, 1>(W, x, xs, T, y, st);
  // long prefills: 128 x 256 tiles (UMMA N = 256, 256 TMEM columns) halve the
  // weight-operand traffic (and, for W4, the dequantisation) per FLOP; FP16 /
  // INT8 run them as CTA pairs (cta_group::2) over adjacent weight-row tiles
  if constexpr (FMT != kW4) {
#ifndef MSW_GEMM_NO_PAIR  // A/B builds only
    if ((W.n / kTileM) % 2 == 0) return launch_bn<FMT, 256, EPI, 2>(W, x, xs, T, y, st);
#endif
  }
  return launch_bn<FMT, 256, EPI, 1>(W, x, xs, T, y, st);
}

template <int FMT>
void launch_fmt(const LinearW& W, int epi, const void* x, const float* xs, int T, float* y,
                cudaStream_t st) {
  if (epi == kEpiStore) return launch_fmt_epi<FMT, kEpiStore>(W, x, xs, T, y, st);
  if (epi == kEpiResid) return launch_fmt_epi<FMT, kEpiResid>(W, x, xs, T, y, st);
  if (epi == kEpiSwiglu) return launch_fmt_epi<FMT, kEpiSwiglu>(W, x, xs, T, y, st);
  if constexpr (FMT == kINT8) {
    if (epi == kEpiRaw) return launch_fmt_epi<FMT, kEpiRaw>(W, x, xs, T, y, st);
  }
  throw ConfigErr("gemm_tc: bad epilogue for this format");
}

}  // namespace

bool gemm_tc_supported(const LinearW& W) {
  return W.n % kTileM == 0 && W.k % 128 == 0 && W.n > 0;
}

void launch_gemm_tc(const LinearW& W, int epi, const half* xh, const int8_t* xq,
                    const float* xscale, int T, float* y, cudaStream_t st) {
  if (!gemm_tc_supported(W)) throw ConfigErr("gemm_tc: n must be a multiple of 128, k of 128");
  switch (W.fmt) {
    case kFP16: return launch_fmt<kFP16>(W, epi, xh, xscale, T, y, st);
    case kINT8: return launch_fmt<kINT8>(W, epi, xq, xscale, T, y, st);
    case kW4: return launch_fmt<kW4>(W, epi, xh, xscale, T, y, st);
    default: throw ConfigErr("gemm_tc: bad format");
  }
}

}  // namespace msw
