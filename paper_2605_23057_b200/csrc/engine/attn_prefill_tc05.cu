// Prefill attention on the 5th-generation tensor cores (tcgen05 + TMEM + TMA)
// for head_dim 128 (the Llama-3.1-8B target): FlashAttention-style, causal,
// over the paged KV cache, with the same packed-window semantics as the
// mma.sync kernel in attn_prefill.cu (token t of sequence seq_of[t] at
// position pos[t] attends to positions [0, pos[t]] of its sequence through
// block_table; a window may hold tokens of several sequences, which are walked
// one after the other with the rows of the others masked).
//
// Per CTA: 128 query rows = 128/G consecutive tokens x the G query heads of
// one kv head (TMEM lane = row), KV tiles of 128 positions.
//   warp 8 (one lane) : TMA producer. A KV tile is 8 paged blocks; each block
//                       is 16 rows x 256 B per kv head, loaded as two
//                       SWIZZLE_128B boxes (d 0..63, 64..127) for K and for V
//                       into a double-buffered ring.
//   warp 9 (one lane) : MMA issuer. S_j = Q K_j^T (kind::f16, M = N = 128,
//                       K = D; Q and K K-major) into one of two TMEM S
//                       buffers, issued one tile ahead of the softmax; then
//                       O += P_j V_j with P (fp16) read from TMEM as the A
//                       operand and V_j as an MN-major B operand (the cache
//                       rows are d-contiguous), accumulating in TMEM.
//   warps 0-7         : softmax, two threads per query row (warps w and w+4
//                       share TMEM lane quarter w & 3 and take the two
//                       64-column halves): tcgen05.ld of the half-row's
//                       scores, one shared-memory exchange of the row max,
//                       causal mask, online softmax in the exp2 domain, the
//                       O rescale (tcgen05.ld/st) and P (tcgen05.st); at the
//                       end O / l -> fp32 o.
// TMEM: S0 [0,128), S1 [128,256), P [256,320) (fp16 pairs), O [320,448).
// Numerics as the mma.sync kernel: fp32 scores of fp16 q / K, P rounded to
// fp16 for the PV product, fp32 accumulation.
#include <cuda.h>

#include <climits>
#include <mutex>
#include <unordered_map>

#include "kernels.cuh"

namespace msw {
namespace {

constexpr int kD = 128;
constexpr int kRows = 128;          // query rows per CTA (UMMA M)
constexpr int kKT = 128;            // KV positions per tile (UMMA N of S, K of PV)
constexpr int kHalfBytes = kKT * 128;         // one 64-d half of a K or V tile (16 KB)
constexpr int kTileBytes = 2 * kHalfBytes;    // K or V tile (32 KB)
constexpr int kQBytes = 2 * kRows * 128;      // Q tile, two 64-d halves (32 KB)
constexpr int kSmem = kQBytes + 2 * 2 * kTileBytes + 1024;  // Q + 2 stages x (K, V) + align
constexpr int kSmWarps = 8;                    // softmax warps: 2 per TMEM lane quarter
constexpr int kThreads = (kSmWarps + 2) * 32;  // + TMA producer + MMA issuer
constexpr int kWProd = kSmWarps, kWMma = kSmWarps + 1;
constexpr uint32_t kColS0 = 0, kColS1 = 128, kColP = 256, kColO = 320;

__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// SWIZZLE_128B descriptors. K-major (Q, K): 8-row x 128 B atoms, SBO = 1024 B.
// MN-major (V): atoms of 8 K-rows (positions) x 64 MN elements (d), SBO =
// 1024 B between 8-position groups, LBO = 16 KB between the two 64-d halves.
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo_bytes) {
  uint64_t d = uint64_t((saddr & 0x3FFFF) >> 4);
  d |= uint64_t((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= uint64_t(1024 >> 4) << 32;
  d |= uint64_t(1) << 46;   // sm_100 descriptor version
  d |= uint64_t(2) << 61;   // SWIZZLE_128B
  return d;
}
// kind::f16, fp16 A / B, fp32 D, M = 128, N = 128; b_mn: B MN-major
__device__ __forceinline__ constexpr uint32_t idesc(bool b_mn) {
  return (1u << 4) | (b_mn ? (1u << 16) : 0u) | (uint32_t(128 >> 3) << 17) | (uint32_t(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tst32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
      "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
      "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tst_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

template <int G>
__global__ void __launch_bounds__(kThreads, 1)
    attn_prefill_tc05_kernel(const __grid_constant__ CUtensorMap tmK,
                             const __grid_constant__ CUtensorMap tmV, const half* __restrict__ q,
                             int T, const int* __restrict__ pos, const int* __restrict__ seq_of,
                             const int* __restrict__ block_table, int max_blocks, int Hq, int Hk,
                             float* __restrict__ o) {
  constexpr int TOK = kRows / G;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                      // [2 halves][128 rows][128 B]
  uint8_t* sKV = smem + kQBytes;           // [stage][K | V][2 halves][128 pos][128 B]
  __shared__ uint64_t kv_full[2], kv_empty[2], s_full[2], p_ready, o_done, q_ready;
  __shared__ uint32_t tmem_slot;
  __shared__ int s_pos[TOK], s_seq[TOK];
  __shared__ float xmax[2][2][kRows];  // [tile parity][column half][row]: partial row maxima
  __shared__ float xl[2][kRows];       // per column half: partial row sums (epilogue)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t0 = blockIdx.x * TOK, hk = blockIdx.y;
  const float sl2 = rsqrtf(float(kD)) * 1.4426950408889634f;  // softmax scale, log2 domain

  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
      mbar_init(&s_full[s], 1);
    }
    mbar_init(&p_ready, kSmWarps);  // one arrive per softmax warp
    mbar_init(&o_done, 1);
    mbar_init(&q_ready, kSmWarps);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmK) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmV) : "memory");
  }
  if (warp == kWMma) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  pdl_wait();
  pdl_trigger();
  for (int i = threadIdx.x; i < TOK; i += blockDim.x) {
    const bool v = t0 + i < T;
    s_pos[i] = v ? pos[t0 + i] : -1;
    s_seq[i] = v ? seq_of[t0 + i] : INT_MAX;
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = tmem_slot;

  // The pass structure (distinct sequences of the window, their causal KV
  // extent) is computed identically by every role from s_pos / s_seq.
  auto next_seq = [&](int prev, int& kv_end, int& lim_max) {
    int nxt = INT_MAX;
    for (int i = 0; i < TOK; ++i)
      if (s_seq[i] > prev && s_seq[i] < nxt) nxt = s_seq[i];
    kv_end = 0;
    for (int i = 0; i < TOK; ++i)
      if (s_seq[i] == nxt) kv_end = max(kv_end, s_pos[i] + 1);
    lim_max = kv_end - 1;
    return nxt;
  };

  if (warp == kWProd) {
    // ---- TMA producer: K and V tiles of every pass, double buffered
    if (lane == 0) {
      int it = 0, seq = INT_MIN, kv_end, lim;
      while ((seq = next_seq(seq, kv_end, lim)) != INT_MAX) {
        const int* bt = block_table + size_t(seq) * max_blocks;
        const int nblk_seq = (kv_end + kKvBlock - 1) / kKvBlock;
        const int ntiles = (kv_end + kKT - 1) / kKT;
        for (int j = 0; j < ntiles; ++j, ++it) {
          const int s = it & 1;
          mbar_wait(&kv_empty[s], ((it >> 1) & 1) ^ 1);
          mbar_expect_tx(&kv_full[s], 2 * kTileBytes);
          uint8_t* dk = sKV + s * 2 * kTileBytes;
          uint8_t* dv = dk + kTileBytes;
          for (int b = 0; b < kKT / kKvBlock; ++b) {
            // blocks past the sequence's extent re-read its first block:
            // finite data under a zero P
            const int lb = j * (kKT / kKvBlock) + b;
            const int blk = bt[lb < nblk_seq ? lb : 0];
            const int row = (blk * Hk + hk) * kKvBlock;
            for (int h = 0; h < 2; ++h) {
              tma2d(dk + h * kHalfBytes + b * kKvBlock * 128, &tmK, &kv_full[s], h * 64, row);
              tma2d(dv + h * kHalfBytes + b * kKvBlock * 128, &tmV, &kv_full[s], h * 64, row);
            }
          }
        }
      }
    }
  } else if (warp == kWMma) {
    // ---- MMA issuer
    if (lane == 0) {
      mbar_wait(&q_ready, 0);
      tc_after();
      const uint32_t qa = smem_u32(sQ);
      // per tile: S_{j} issued one tile ahead of PV_{j-1}
      int it = 0, seq = INT_MIN, kv_end, lim;
      int pv_done = 0;  // PV tiles issued
      auto issue_s = [&](int j_it) {
        const int s = j_it & 1;
        mbar_wait(&kv_full[s], (j_it >> 1) & 1);
        tc_after();
        const uint32_t kb = smem_u32(sKV + s * 2 * kTileBytes);
#pragma unroll
        for (int k = 0; k < kD / 16; ++k) {  // K = D in 16-element steps, two 64-d halves
          const uint32_t off = (k >> 2) * kHalfBytes + (k & 3) * 32;
          mma_ss(tmem + (s ? kColS1 : kColS0), desc_sw128(qa + (k >> 2) * (kRows * 128) + (k & 3) * 32, 16),
                 desc_sw128(kb + off, 16), idesc(false), k != 0);
        }
        commit(&s_full[s]);
      };
      auto issue_pv = [&](int j_it) {
        const int s = j_it & 1;
        mbar_wait(&p_ready, j_it & 1);
        tc_after();
        const uint32_t vb = smem_u32(sKV + s * 2 * kTileBytes + kTileBytes);
#pragma unroll
        for (int k = 0; k < kKT / 16; ++k)  // K = positions, 16 per step (2048 B of V rows)
          mma_ts(tmem + kColO, tmem + kColP + k * 8, desc_sw128(vb + k * 2048, kHalfBytes),
                 idesc(true), (j_it | k) != 0);
        commit(&o_done);
        commit(&kv_empty[s]);
      };
      while ((seq = next_seq(seq, kv_end, lim)) != INT_MAX) {
        const int ntiles = (kv_end + kKT - 1) / kKT;
        for (int j = 0; j < ntiles; ++j, ++it) {
          issue_s(it);
          if (it > 0) issue_pv(it - 1);
          pv_done = it;
        }
      }
      if (it > 0) issue_pv(it - 1);
      (void)pv_done;
    }
  } else {
    // ---- softmax / epilogue warps 0-7: thread = (query row r = tl * G + g,
    // column half ch); warps w and w + 4 share TMEM lane quarter w & 3
    const int r = (warp & 3) * 32 + lane, ch = warp >> 2;
    const int tl = r / G, g = r % G;
    const int t = t0 + tl;
    const int hq = hk * G + g;
    {  // Q row half -> SW128 K-major smem (64-d half ch), 16-byte chunks XOR (r & 7)
      const uint4* src = reinterpret_cast<const uint4*>(q + (size_t(t < T ? t : 0) * Hq + hq) * kD) + ch * 8;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint4 v = t < T ? src[c] : make_uint4(0, 0, 0, 0);
        *reinterpret_cast<uint4*>(sQ + ch * (kRows * 128) + r * 128 + ((c ^ (r & 7)) << 4)) = v;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&q_ready);
    }
    const uint32_t trow = tmem + (uint32_t((warp & 3) * 32) << 16);
    const uint32_t col_s = ch * 64, col_p = ch * 32, col_o = ch * 64;
    const int my_pos = s_pos[tl], my_seq = s_seq[tl];
    float m = -INFINITY, l = 0.0f;  // l: this half's partial sum (same scale as the other half)
    int it = 0, seq = INT_MIN, kv_end, lim_max;
    while ((seq = next_seq(seq, kv_end, lim_max)) != INT_MAX) {
      const int lim = my_seq == seq ? my_pos : -1;
      const int ntiles = (kv_end + kKT - 1) / kKT;
      for (int j = 0; j < ntiles; ++j, ++it) {
        const int s = it & 1;
        mbar_wait(&s_full[s], (it >> 1) & 1);
        tc_after();
        // this half's 64 scores of the row
        float sc[64];
#pragma unroll
        for (int c2 = 0; c2 < 2; ++c2) {
          uint32_t u[32];
          tld32(trow + (s ? kColS1 : kColS0) + col_s + c2 * 32, u);
          tld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) sc[c2 * 32 + i] = __uint_as_float(u[i]);
        }
        float mt = -INFINITY;
#pragma unroll
        for (int i = 0; i < 64; ++i) {
          const int kp = j * kKT + ch * 64 + i;
          sc[i] = kp <= lim ? sc[i] * sl2 : -INFINITY;
          mt = fmaxf(mt, sc[i]);
        }
        // row maximum over both halves (double-buffered exchange: one barrier per tile)
        xmax[s][ch][r] = mt;
        named_sync(2, kSmWarps * 32);
        mt = fmaxf(mt, xmax[s][ch ^ 1][r]);
        const float mn = fmaxf(m, mt);
        const float u0 = mn == -INFINITY ? 0.0f : mn;
        const float corr = exp2f(m - u0);
        m = mn;
        float ls = 0.0f;
        uint32_t pk[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float e0 = exp2f(sc[2 * i] - u0), e1 = exp2f(sc[2 * i + 1] - u0);
          ls += e0 + e1;
          const half2 h = __floats2half2_rn(e0, e1);
          pk[i] = *reinterpret_cast<const uint32_t*>(&h);
        }
        l = l * corr + ls;
        // PV of the previous tile must be complete before O is rescaled and P overwritten
        if (it > 0) {
          mbar_wait(&o_done, (it - 1) & 1);
          tc_after();
          // rescale this half of O only when some row of the warp saw a new
          // maximum (the row maxima settle after the first tiles)
          if (__any_sync(0xffffffffu, corr != 1.0f))
#pragma unroll
          for (int c2 = 0; c2 < 2; ++c2) {
            uint32_t u[32];
            tld32(trow + kColO + col_o + c2 * 32, u);
            tld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) u[i] = __float_as_uint(__uint_as_float(u[i]) * corr);
            tst32(trow + kColO + col_o + c2 * 32, u);
          }
        }
        tst32(trow + kColP + col_p, pk);
        tst_wait();
        tc_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_ready);
      }
    }
    // epilogue: O / l, l = both halves' partial sums
    xl[ch][r] = l;
    if (it > 0) {
      mbar_wait(&o_done, (it - 1) & 1);
      tc_after();
    }
    named_sync(2, kSmWarps * 32);
    const float lt = l + xl[ch ^ 1][r];
    const float inv = lt > 0.0f ? 1.0f / lt : 0.0f;
#pragma unroll
    for (int c2 = 0; c2 < 2; ++c2) {
      uint32_t u[32];
      tld32(trow + kColO + col_o + c2 * 32, u);
      tld_wait();
      if (t < T && it > 0) {
        float4* dst = reinterpret_cast<float4*>(o + (size_t(t) * Hq + hq) * kD + col_o + c2 * 32);
#pragma unroll
        for (int i = 0; i < 8; ++i)
          dst[i] = make_float4(__uint_as_float(u[4 * i]) * inv, __uint_as_float(u[4 * i + 1]) * inv,
                               __uint_as_float(u[4 * i + 2]) * inv, __uint_as_float(u[4 * i + 3]) * inv);
      }
    }
  }
  tc_before();
  __syncthreads();
  if (warp == kWMma)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

EncodeFn encode() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) != cudaSuccess ||
        qr != cudaDriverEntryPointSuccess)
      p = nullptr;
    fn = reinterpret_cast<EncodeFn>(p);
  });
  if (!fn) throw CudaError("cuTensorMapEncodeTiled unavailable");
  return fn;
}

// One layer's K (or V) cache viewed as [rows = blocks * Hk * 16][128] fp16,
// boxes of 16 rows x 64 d with SWIZZLE_128B. Cached per base pointer.
const CUtensorMap& kv_map(const half* base, uint64_t rows) {
  static std::unordered_map<const void*, CUtensorMap> cache;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(base);
  if (it != cache.end()) return it->second;
  CUtensorMap m;
  const cuuint64_t dims[2] = {uint64_t(kD), rows};
  const cuuint64_t strides[1] = {uint64_t(kD) * 2};
  const cuuint32_t box[2] = {64, uint32_t(kKvBlock)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<half*>(base), dims, strides,
                              box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (kv) failed: " + std::to_string(int(r)));
  return cache.emplace(base, m).first->second;
}

template <int G>
void launch_g(int T, const half* q, const int* pos, const int* seq_of, const int* bt, int maxb,
              const half* kc, const half* vc, uint64_t kv_rows, int Hq, int Hk, float* o,
              cudaStream_t st) {
  constexpr int TOK = kRows / G;
  static bool attr = false;
  if (!attr) {
    MSW_CUDA(cudaFuncSetAttribute(attn_prefill_tc05_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kSmem));
    attr = true;
  }
  const CUtensorMap mk = kv_map(kc, kv_rows), mv = kv_map(vc, kv_rows);
  launch_pdl(attn_prefill_tc05_kernel<G>, dim3((T + TOK - 1) / TOK, Hk), dim3(kThreads), kSmem, st, mk,
             mv, q, T, pos, seq_of, bt, maxb, Hq, Hk, o);
}

}  // namespace

bool attention_prefill_tc05_supported(const AttnShape& a) {
  const int G = a.n_heads / a.n_kv_heads;
  return a.head_dim == kD && (G == 1 || G == 2 || G == 4 || G == 8);
}

void launch_attention_prefill_tc05(const half* q, int T, const int* pos, const int* seq_of,
                                   const int* block_table, const half* kc, const half* vc,
                                   uint64_t kv_rows, const AttnShape& a, float* o, cudaStream_t st) {
  const int G = a.n_heads / a.n_kv_heads;
  switch (G) {
    case 1: return launch_g<1>(T, q, pos, seq_of, block_table, a.max_blocks_per_seq, kc, vc, kv_rows, a.n_heads, a.n_kv_heads, o, st);
    case 2: return launch_g<2>(T, q, pos, seq_of, block_table, a.max_blocks_per_seq, kc, vc, kv_rows, a.n_heads, a.n_kv_heads, o, st);
    case 4: return launch_g<4>(T, q, pos, seq_of, block_table, a.max_blocks_per_seq, kc, vc, kv_rows, a.n_heads, a.n_kv_heads, o, st);
    case 8: return launch_g<8>(T, q, pos, seq_of, block_table, a.max_blocks_per_seq, kc, vc, kv_rows, a.n_heads, a.n_kv_heads, o, st);
    default: throw ConfigErr("attention (tc05): GQA group must be 1, 2, 4 or 8");
  }
}

}  // namespace msw
