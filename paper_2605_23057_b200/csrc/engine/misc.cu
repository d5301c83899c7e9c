// Embedding gather, greedy argmax and the device-side decode bookkeeping that
// lets a whole batch-1 decode step replay from a CUDA graph with no host sync.
#include "kernels.cuh"

namespace msw {
namespace {

__global__ void embed_kernel(const half* __restrict__ emb, const int* __restrict__ tok, int H,
                             float* __restrict__ h) {
  pdl_wait();
  pdl_trigger();
  const int t = blockIdx.x;
  const half* row = emb + size_t(tok[t]) * H;
  for (int i = threadIdx.x; i < H; i += blockDim.x) h[size_t(t) * H + i] = __half2float(row[i]);
}

// Lowest index wins ties: compare (value, -index) lexicographically.
__device__ __forceinline__ void better(float& bv, int& bi, float v, int i) {
  if (v > bv || (v == bv && i < bi)) {
    bv = v;
    bi = i;
  }
}

// Multi-CTA greedy argmax: grid (blocks, T). Every CTA reduces a slice of the
// row to one (value, index) key, folds it into slot[t] with a 64-bit
// atomicMax, and the last CTA of the row (counter) publishes the index and
// resets slot / counter for the next step. Key = order-preserving fp32 bits
// in the high word, ~index in the low word, so equal values resolve to the
// lowest index.
constexpr int kArgmaxThreads = 256;
constexpr int kArgmaxPerCta = 4096;

__device__ __forceinline__ unsigned long long amax_key(float v, int i) {
  const uint32_t u = __float_as_uint(v);
  const uint32_t o = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return (static_cast<unsigned long long>(o) << 32) | (0xFFFFFFFFu - uint32_t(i));
}

__global__ void __launch_bounds__(kArgmaxThreads)
    argmax_kernel(const float* __restrict__ logits, int V, int* __restrict__ out,
                  unsigned long long* __restrict__ slot, int* __restrict__ cnt) {
  __shared__ unsigned long long sk[kArgmaxThreads / 32];
  __shared__ int is_last;
  pdl_wait();
  pdl_trigger();
  const int t = blockIdx.y;
  const float* row = logits + size_t(t) * V;
  const int b0 = blockIdx.x * kArgmaxPerCta;
  const int b1 = min(V, b0 + kArgmaxPerCta);
  unsigned long long best = 0;
  for (int i = b0 + threadIdx.x; i < b1; i += kArgmaxThreads) {
    const unsigned long long kk = amax_key(__ldcg(row + i), i);
    best = kk > best ? kk : best;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long ok = __shfl_xor_sync(0xffffffffu, best, o);
    best = ok > best ? ok : best;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sk[warp] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kArgmaxThreads / 32; ++w) best = sk[w] > best ? sk[w] : best;
    atomicMax(slot + t, best);
    __threadfence();
    is_last = atomicAdd(cnt + t, 1) == int(gridDim.x) - 1;
    if (is_last) {
      __threadfence();
      const unsigned long long k = atomicExch(slot + t, 0ull);
      cnt[t] = 0;
      out[t] = int(0xFFFFFFFFu - uint32_t(k & 0xFFFFFFFFull));
    }
  }
}

__global__ void gather_rows_kernel(const float* __restrict__ src, const int* __restrict__ rows,
                                   int width, float* __restrict__ dst) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x;
  const float* s = src + size_t(rows[r]) * width;
  for (int i = threadIdx.x; i < width; i += blockDim.x) dst[size_t(r) * width + i] = s[i];
}

// Batch-1 decode bookkeeping: the argmax output becomes the next input token,
// is appended to the device-resident history, and the position/slot advance
// through block-table row 0.
__global__ void advance_kernel(const int* next, int* tok, int* pos, int* slot, int* step,
                               int* history, const int* block_table) {
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x != 0) return;
  const int s = step[0];
  const int t = next[0];
  history[s] = t;
  tok[0] = t;
  step[0] = s + 1;
  const int p = pos[0] + 1;
  pos[0] = p;
  slot[0] = block_table[p >> 4] * kKvBlock + (p & 15);
}

}  // namespace

void launch_embed(const half* emb, const int* tok, int T, int H, float* h, cudaStream_t st) {
  launch_pdl(embed_kernel, dim3(T), dim3(256), 0, st, emb, tok, H, h);
}

void launch_argmax(const float* logits, int T, int V, int* out, unsigned long long* ws,
                   cudaStream_t st) {
  launch_pdl(argmax_kernel, dim3(ceil_div(V, kArgmaxPerCta), T), dim3(kArgmaxThreads), 0, st,
             logits, V, out, ws, reinterpret_cast<int*>(ws + T));
}

void launch_gather_rows(const float* src, const int* rows, int n, int width, float* dst,
                        cudaStream_t st) {
  launch_pdl(gather_rows_kernel, dim3(n), dim3(256), 0, st, src, rows, width, dst);
}

void launch_advance(const int* next, int* tok, int* pos, int* slot, int* step, int* history,
                    const int* block_table, cudaStream_t st) {
  launch_pdl(advance_kernel, dim3(1), dim3(32), 0, st, next, tok, pos, slot, step, history,
             block_table);
}

}  // namespace msw
