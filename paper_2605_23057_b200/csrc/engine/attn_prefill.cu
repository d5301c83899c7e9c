// Tensor-core prefill attention over the paged KV cache (FlashAttention-2
// style, mma.sync m16n8k16 f16 -> f32), for forward passes with many query
// tokens (prefill chunks, packed continuous-batching admissions).
//
// Semantics are those of launch_attention (attention.cu): token t of sequence
// seq_of[t] at position pos[t] attends to positions [0, pos[t]] of its
// sequence through block_table[seq_of[t]] (causal; prefix-cache hits are just
// shared physical blocks). Tokens may be packed from several sequences in any
// order: a CTA owns a window of TOK consecutive query tokens x the G query
// heads of one kv head (128 rows, 8 warps x 16 rows) and walks the KV of every
// distinct sequence present in its window, rows of other sequences masked.
//
// Per KV tile (64 positions): K and V rows are gathered from 16-token paged
// blocks by cp.async into XOR-swizzled shared memory (double-buffered), B
// fragments come from ldmatrix (.trans for V), S = Q K^T and O += P V run on
// the tensor pipe, the online softmax stays in registers (exp2 domain). The
// reference (sim.cpp:80-145) has no kernel here: the numerics follow the
// oracle's fp32 attention over fp16 q / K / V; P is rounded to fp16 for the
// PV product (the tests' FP16 logit tolerance covers it).
#include <climits>

#include "kernels.cuh"

namespace msw {
namespace {

constexpr int kPfWarps = 8;
constexpr int kPfRows = kPfWarps * 16;  // query rows (token x head) per CTA
constexpr int kPfKT = 64;               // kv positions per tile

__device__ __forceinline__ size_t kv_off_pf(int slot, int hk, int Hk, int D) {
  return ((size_t(slot >> 4) * Hk + hk) * kKvBlock + (slot & 15)) * size_t(D);
}

__device__ __forceinline__ void cp_async16_zfill(void* smem_dst, const void* gsrc, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem_dst)),
               "l"(gsrc), "r"(valid ? 16 : 0)
               : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
  const half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// row r, 16-byte chunk c of a [rows][D] fp16 tile, XOR-swizzled so the 8 rows
// an ldmatrix phase reads land in 8 distinct bank groups
template <int D>
__device__ __forceinline__ int swz(int r, int c) {
  return r * D + ((c ^ (r & 7)) << 3);
}

template <int D, int G>
__global__ void __launch_bounds__(kPfWarps * 32, 1)
    attn_prefill_tc_kernel(const half* __restrict__ q, int T, const int* __restrict__ pos,
                           const int* __restrict__ seq_of, const int* __restrict__ block_table,
                           int max_blocks, const half* __restrict__ kc,
                           const half* __restrict__ vc, int Hq, int Hk, float* __restrict__ o) {
  constexpr int TOK = kPfRows / G;  // query tokens per CTA
  constexpr int CH = D / 8;         // 16-byte chunks per K/V row
  constexpr int NT = kPfKT / 8;     // score n-tiles per KV tile
  constexpr int DT = D / 8;         // output n-tiles
  extern __shared__ __align__(128) uint8_t pf_smem[];
  half* sK = reinterpret_cast<half*>(pf_smem);  // [2][KT][D]
  half* sV = sK + 2 * kPfKT * D;                // [2][KT][D]
  __shared__ int s_pos[TOK], s_seq[TOK];

  const int t0 = blockIdx.x * TOK, hk = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = warp % G;               // query head within the group
  const int tw = (warp / G) * 16;       // first token row of this warp
  const int hq = hk * G + g;
  const float sl2 = rsqrtf(float(D)) * 1.4426950408889634f;  // softmax scale, log2 domain

  pdl_wait();
  pdl_trigger();
  for (int i = threadIdx.x; i < TOK; i += blockDim.x) {
    const bool v = t0 + i < T;
    s_pos[i] = v ? pos[t0 + i] : -1;
    s_seq[i] = v ? seq_of[t0 + i] : INT_MAX;
  }
  __syncthreads();

  // Q fragments (A operand, row-major 16 x D): rows lane/4 and lane/4 + 8
  const int ra = tw + (lane >> 2), rb = ra + 8;
  uint32_t qf[D / 16][4];
#pragma unroll
  for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int row = (r & 1) ? rb : ra;
      const int col = kk * 16 + (lane & 3) * 2 + ((r & 2) ? 8 : 0);
      const int t = t0 + row;
      qf[kk][r] = t < T ? *reinterpret_cast<const uint32_t*>(q + (size_t(t) * Hq + hq) * D + col)
                        : 0u;
    }
  }
  const int pa = s_pos[ra], pb = s_pos[rb];
  const int qa = s_seq[ra], qb = s_seq[rb];

  float oacc[DT][4];
#pragma unroll
  for (int i = 0; i < DT; ++i) oacc[i][0] = oacc[i][1] = oacc[i][2] = oacc[i][3] = 0.0f;
  float ma = -INFINITY, mb = -INFINITY, la = 0.0f, lb = 0.0f;

  const uint32_t sK_u = smem_u32(sK), sV_u = smem_u32(sV);
  int seq = INT_MIN;
  while (true) {
    // next distinct sequence of this window (ascending id), its KV extent
    int nxt = INT_MAX, kv_end = 0;
    for (int i = 0; i < TOK; ++i) {
      const int sq = s_seq[i];
      if (sq > seq && sq < nxt) nxt = sq;
    }
    if (nxt == INT_MAX) break;
    seq = nxt;
    for (int i = 0; i < TOK; ++i)
      if (s_seq[i] == seq) kv_end = max(kv_end, s_pos[i] + 1);
    const int lim_a = qa == seq ? pa : -1, lim_b = qb == seq ? pb : -1;
    int warp_lim = max(lim_a, lim_b);
    warp_lim = max(warp_lim, __shfl_xor_sync(0xffffffffu, warp_lim, 1));
    warp_lim = max(warp_lim, __shfl_xor_sync(0xffffffffu, warp_lim, 2));
    warp_lim = max(warp_lim, __shfl_xor_sync(0xffffffffu, warp_lim, 4));
    warp_lim = max(warp_lim, __shfl_xor_sync(0xffffffffu, warp_lim, 8));
    warp_lim = max(warp_lim, __shfl_xor_sync(0xffffffffu, warp_lim, 16));
    const int* bt = block_table + size_t(seq) * max_blocks;
    const int ntiles = (kv_end + kPfKT - 1) / kPfKT;

    auto load_tile = [&](int j, int stage) {
      half* dk = sK + stage * kPfKT * D;
      half* dv = sV + stage * kPfKT * D;
      for (int idx = threadIdx.x; idx < kPfKT * CH; idx += blockDim.x) {
        const int r = idx / CH, c = idx % CH;
        const int p = j * kPfKT + r;
        const bool ok = p < kv_end;
        const size_t off = ok ? kv_off_pf(bt[p >> 4] * kKvBlock + (p & 15), hk, Hk, D) + c * 8 : 0;
        cp_async16_zfill(dk + swz<D>(r, c), kc + off, ok);
        cp_async16_zfill(dv + swz<D>(r, c), vc + off, ok);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };

    load_tile(0, 0);
    for (int j = 0; j < ntiles; ++j) {
      if (j + 1 < ntiles) {
        load_tile(j + 1, (j + 1) & 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncthreads();
      const int kbase = j * kPfKT;
      if (kbase <= warp_lim) {  // causal: tiles past every row of this warp are skipped
        const uint32_t kst = sK_u + uint32_t((j & 1) * kPfKT * D * 2);
        const uint32_t vst = sV_u + uint32_t((j & 1) * kPfKT * D * 2);
        float s[NT][4];
#pragma unroll
        for (int i = 0; i < NT; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.0f;
        // S = Q K^T
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
          for (int np = 0; np < NT / 2; ++np) {
            const int mi = lane >> 3;
            const int r = np * 16 + (mi >> 1) * 8 + (lane & 7);
            const int c = kk * 2 + (mi & 1);
            uint32_t b0, b1, b2, b3;
            ldsm_x4(kst + uint32_t(swz<D>(r, c) * 2), b0, b1, b2, b3);
            mma16816(s[2 * np], qf[kk], b0, b1);
            mma16816(s[2 * np + 1], qf[kk], b2, b3);
          }
        }
        // mask + online softmax (rows a: s[.][0..1], rows b: s[.][2..3])
        float tma = -INFINITY, tmb = -INFINITY;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int kp = kbase + nt * 8 + (lane & 3) * 2 + (e & 1);
            const int lim = e < 2 ? lim_a : lim_b;
            const float v = kp <= lim ? s[nt][e] * sl2 : -INFINITY;
            s[nt][e] = v;
            if (e < 2) tma = fmaxf(tma, v);
            else tmb = fmaxf(tmb, v);
          }
        }
        tma = fmaxf(tma, __shfl_xor_sync(0xffffffffu, tma, 1));
        tma = fmaxf(tma, __shfl_xor_sync(0xffffffffu, tma, 2));
        tmb = fmaxf(tmb, __shfl_xor_sync(0xffffffffu, tmb, 1));
        tmb = fmaxf(tmb, __shfl_xor_sync(0xffffffffu, tmb, 2));
        const float mna = fmaxf(ma, tma), mnb = fmaxf(mb, tmb);
        const float ua = mna == -INFINITY ? 0.0f : mna, ub = mnb == -INFINITY ? 0.0f : mnb;
        const float ca = exp2f(ma - ua), cb = exp2f(mb - ub);
        ma = mna;
        mb = mnb;
        float sa = 0.0f, sb = 0.0f;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          s[nt][0] = exp2f(s[nt][0] - ua);
          s[nt][1] = exp2f(s[nt][1] - ua);
          s[nt][2] = exp2f(s[nt][2] - ub);
          s[nt][3] = exp2f(s[nt][3] - ub);
          sa += s[nt][0] + s[nt][1];
          sb += s[nt][2] + s[nt][3];
        }
        la = la * ca + sa;
        lb = lb * cb + sb;
#pragma unroll
        for (int i = 0; i < DT; ++i) {
          oacc[i][0] *= ca;
          oacc[i][1] *= ca;
          oacc[i][2] *= cb;
          oacc[i][3] *= cb;
        }
        // O += P V
#pragma unroll
        for (int k2 = 0; k2 < kPfKT / 16; ++k2) {
          uint32_t pa4[4];
          pa4[0] = pack_h2(s[2 * k2][0], s[2 * k2][1]);
          pa4[1] = pack_h2(s[2 * k2][2], s[2 * k2][3]);
          pa4[2] = pack_h2(s[2 * k2 + 1][0], s[2 * k2 + 1][1]);
          pa4[3] = pack_h2(s[2 * k2 + 1][2], s[2 * k2 + 1][3]);
#pragma unroll
          for (int dp = 0; dp < DT / 2; ++dp) {
            const int mi = lane >> 3;
            const int r = k2 * 16 + (mi & 1) * 8 + (lane & 7);
            const int c = dp * 2 + (mi >> 1);
            uint32_t b0, b1, b2, b3;
            ldsm_x4_t(vst + uint32_t(swz<D>(r, c) * 2), b0, b1, b2, b3);
            mma16816(oacc[2 * dp], pa4, b0, b1);
            mma16816(oacc[2 * dp + 1], pa4, b2, b3);
          }
        }
      }
      __syncthreads();  // stage (j & 1) is refilled by the next iteration's load
    }
  }

  // normalise and store (fp32 o[t][hq][d])
  la += __shfl_xor_sync(0xffffffffu, la, 1);
  la += __shfl_xor_sync(0xffffffffu, la, 2);
  lb += __shfl_xor_sync(0xffffffffu, lb, 1);
  lb += __shfl_xor_sync(0xffffffffu, lb, 2);
  const float ia = la > 0.0f ? 1.0f / la : 0.0f, ib = lb > 0.0f ? 1.0f / lb : 0.0f;
  const int ta = t0 + ra, tb = t0 + rb;
#pragma unroll
  for (int i = 0; i < DT; ++i) {
    const int col = i * 8 + (lane & 3) * 2;
    if (ta < T)
      *reinterpret_cast<float2*>(o + (size_t(ta) * Hq + hq) * D + col) =
          make_float2(oacc[i][0] * ia, oacc[i][1] * ia);
    if (tb < T)
      *reinterpret_cast<float2*>(o + (size_t(tb) * Hq + hq) * D + col) =
          make_float2(oacc[i][2] * ib, oacc[i][3] * ib);
  }
}

template <int D, int G>
void launch_pf(int T, const half* q, const int* pos, const int* seq_of, const int* bt, int maxb,
               const half* kc, const half* vc, int Hq, int Hk, float* o, cudaStream_t st) {
  constexpr int TOK = kPfRows / G;
  const size_t smem = size_t(4) * kPfKT * D * sizeof(half);
  static bool attr = false;
  if (!attr) {
    MSW_CUDA(cudaFuncSetAttribute(attn_prefill_tc_kernel<D, G>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr = true;
  }
  launch_pdl(attn_prefill_tc_kernel<D, G>, dim3((T + TOK - 1) / TOK, Hk), dim3(kPfWarps * 32),
             smem, st, q, T, pos, seq_of, bt, maxb, kc, vc, Hq, Hk, o);
}

}  // namespace

void launch_attention_prefill(const half* q, int T, const int* pos, const int* seq_of,
                              const int* block_table, const half* kc, const half* vc,
                              const AttnShape& a, float* o, cudaStream_t st) {
  if (a.n_blocks > 0 && attention_prefill_tc05_supported(a))
    return launch_attention_prefill_tc05(q, T, pos, seq_of, block_table, kc, vc,
                                         uint64_t(a.n_blocks) * a.n_kv_heads * kKvBlock, a, o, st);
  const int G = a.n_heads / a.n_kv_heads;
#define MSW_PF(DD, GG)                                                                       \
  if (a.head_dim == DD && G == GG)                                                           \
    return launch_pf<DD, GG>(T, q, pos, seq_of, block_table, a.max_blocks_per_seq, kc, vc,  \
                             a.n_heads, a.n_kv_heads, o, st);
  MSW_PF(128, 1)
  MSW_PF(128, 2)
  MSW_PF(128, 4)
  MSW_PF(128, 8)
  MSW_PF(64, 1)
  MSW_PF(64, 2)
  MSW_PF(64, 4)
  MSW_PF(64, 8)
#undef MSW_PF
  throw ConfigErr("attention: unsupported head_dim / GQA group");
}

}  // namespace msw
