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

__global__ void argmax_kernel(const float* __restrict__ logits, int V, int* __restrict__ out) {
  __shared__ float sv[32];
  __shared__ int si[32];
  pdl_wait();
  pdl_trigger();
  const int t = blockIdx.x;
  const float* row = logits + size_t(t) * V;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < V; i += blockDim.x) better(bv, bi, row[i], i);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    better(bv, bi, ov, oi);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    sv[warp] = bv;
    si[warp] = bi;
  }
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    bv = lane < nw ? sv[lane] : -INFINITY;
    bi = lane < nw ? si[lane] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      better(bv, bi, ov, oi);
    }
    if (lane == 0) out[t] = bi == 0x7fffffff ? 0 : bi;
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

void launch_argmax(const float* logits, int T, int V, int* out, cudaStream_t st) {
  launch_pdl(argmax_kernel, dim3(T), dim3(1024), 0, st, logits, V, out);
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
