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


// Continuous-batching step bookkeeping (T live sequences, one token each):
// the step's argmax becomes each sequence's next input, is appended to that
// sequence's device history (index hbase[t] + pos[t]), and position / slot
// advance through the sequence's own block-table row (seq_of[t]).
__global__ void cb_advance_kernel(const int* __restrict__ next, int T, int* tok, int* pos,
                                  int* slot, const int* __restrict__ seq_of,
                                  const int* __restrict__ hbase, int* hist,
                                  const int* __restrict__ block_table, int bt_stride) {
  pdl_wait();
  pdl_trigger();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const int out = next[t];
  const int p = pos[t];
  hist[hbase[t] + p] = out;
  tok[t] = out;
  pos[t] = p + 1;
  slot[t] = block_table[size_t(seq_of[t]) * bt_stride + ((p + 1) >> 4)] * kKvBlock + ((p + 1) & 15);
}

// ---- speculative decoding, device side (one round = draft T=2 step, k-1
// draft T=1 steps, target verify of k+1 tokens, accept) --------------------
// Draft step 0 re-runs position n-2 with the token already there (same
// token, same position: the KV it rewrites is the same value up to
// summation order) together with the newest committed token at n-1, so the
// round's shape never depends on how many proposals the previous round
// accepted (the host loop needed a variable-length catch-up after a fully
// accepted round).
__global__ void spec_draft_setup_kernel(const SpecState* __restrict__ ss, int* tok, int* pos,
                                        int* slot, int* seq_of, int* logit_rows,
                                        const int* __restrict__ block_table) {
  pdl_wait();
  pdl_trigger();
  const int t = threadIdx.x;
  if (t >= 2) return;
  const int n = ss->n;
  const int p = n - 2 + t;
  tok[t] = t == 0 ? ss->prev : ss->last;
  pos[t] = p;
  slot[t] = block_table[p >> 4] * kKvBlock + (p & 15);
  seq_of[t] = 0;
  if (t == 0) logit_rows[0] = 1;
}

// proposal i-1 (from the previous draft step's argmax) becomes the input of
// draft step i at position n-1+i
__global__ void spec_draft_next_kernel(SpecState* ss, int i, const int* __restrict__ next,
                                       int* tok, int* pos, int* slot, int* seq_of,
                                       const int* __restrict__ block_table) {
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x != 0) return;
  const int d = next[0];
  ss->props[i - 1] = d;
  const int p = ss->n - 1 + i;
  tok[0] = d;
  pos[0] = p;
  slot[0] = block_table[p >> 4] * kKvBlock + (p & 15);
  seq_of[0] = 0;
}

// target verify input: [last, d_1 .. d_k] at positions n-1 .. n-1+k
__global__ void spec_verify_setup_kernel(SpecState* ss, int k, const int* __restrict__ next,
                                         int* tok, int* pos, int* slot, int* seq_of,
                                         const int* __restrict__ block_table) {
  pdl_wait();
  pdl_trigger();
  const int t = threadIdx.x;
  if (t > k) return;
  if (t == k) ss->props[k - 1] = next[0];  // the last draft step's argmax
  const int d = t == 0 ? ss->last : (t == k ? next[0] : ss->props[t - 1]);
  const int p = ss->n - 1 + t;
  tok[t] = d;
  pos[t] = p;
  slot[t] = block_table[p >> 4] * kKvBlock + (p & 15);
  seq_of[t] = 0;
}

// Accept the longest prefix where the target's greedy token equals the
// draft's proposal, plus the target's own next token; emitted tokens are
// appended to the request's output. Single thread: k <= 8 compares. With
// `cond` the enclosing WHILE node's condition becomes "tokens still to emit".
__device__ __forceinline__ int spec_matched(const SpecState* ss, int k, const int* g) {
  int j = 0;
  while (j < k && ss->props[j] == g[j]) ++j;
  return j;
}

// Logits rows of the tokens this round will emit -> the request's logits
// output (only when requested). Runs BEFORE spec_accept_kernel and reads the
// state without modifying it, so all CTAs see the same round.
__global__ void spec_copy_logits_kernel(const SpecState* __restrict__ ss, int k,
                                        const int* __restrict__ g,
                                        const float* __restrict__ logits, int V) {
  pdl_wait();
  pdl_trigger();
  float* lg = ss->logits_out;
  if (!lg) return;
  const int j = spec_matched(ss, k, g);
  const int emitted = ss->emitted;
  const int ne = min(j + 1, ss->n_new - emitted);
  const long long total = (long long)ne * V;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x)
    lg[(long long)emitted * V + i] = logits[i];
}

__global__ void spec_accept_kernel(SpecState* ss, int k, const int* __restrict__ g,
                                   cudaGraphConditionalHandle cond, int use_cond) {
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x != 0) return;
  const int j = spec_matched(ss, k, g);
  const int emitted = ss->emitted;
  const int ne = min(j + 1, ss->n_new - emitted);  // committed this round: g[0 .. ne-1]
  for (int i = 0; i < ne; ++i) ss->out[emitted + i] = g[i];
  ss->prev = ne >= 2 ? g[ne - 2] : ss->last;
  ss->last = g[ne - 1];
  ss->n += ne;
  ss->emitted = emitted + ne;
  ss->rounds += 1;
  ss->proposed += k;
  ss->accepted += j;
  if (use_cond) cudaGraphSetConditional(cond, emitted + ne < ss->n_new ? 1u : 0u);
}

// first token (target prefill argmax) -> state
__global__ void spec_init_kernel(SpecState* ss, const int* __restrict__ next, int plen, int n_new,
                                 int prompt_last, float* logits_out) {
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x != 0) return;
  const int t = next[0];
  ss->n = plen + 1;
  ss->prev = prompt_last;
  ss->last = t;
  ss->emitted = 1;
  ss->n_new = n_new;
  ss->rounds = ss->proposed = ss->accepted = 0;
  ss->out[0] = t;
  ss->logits_out = logits_out;
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

void launch_cb_advance(const int* next, int T, int* tok, int* pos, int* slot, const int* seq_of,
                       const int* hbase, int* hist, const int* block_table, int bt_stride,
                       cudaStream_t st) {
  launch_pdl(cb_advance_kernel, dim3(ceil_div(T, 64)), dim3(64), 0, st, next, T, tok, pos, slot,
             seq_of, hbase, hist, block_table, bt_stride);
}

void launch_spec_init(SpecState* ss, const int* next, int plen, int n_new, int prompt_last,
                      float* logits_out, cudaStream_t st) {
  launch_pdl(spec_init_kernel, dim3(1), dim3(32), 0, st, ss, next, plen, n_new, prompt_last,
             logits_out);
}

void launch_spec_draft_setup(const SpecState* ss, int* tok, int* pos, int* slot, int* seq_of,
                             int* logit_rows, const int* block_table, cudaStream_t st) {
  launch_pdl(spec_draft_setup_kernel, dim3(1), dim3(32), 0, st, ss, tok, pos, slot, seq_of,
             logit_rows, block_table);
}

void launch_spec_draft_next(SpecState* ss, int i, const int* next, int* tok, int* pos, int* slot,
                            int* seq_of, const int* block_table, cudaStream_t st) {
  launch_pdl(spec_draft_next_kernel, dim3(1), dim3(32), 0, st, ss, i, next, tok, pos, slot, seq_of,
             block_table);
}

void launch_spec_verify_setup(SpecState* ss, int k, const int* next, int* tok, int* pos, int* slot,
                              int* seq_of, const int* block_table, cudaStream_t st) {
  launch_pdl(spec_verify_setup_kernel, dim3(1), dim3(32), 0, st, ss, k, next, tok, pos, slot,
             seq_of, block_table);
}

void launch_spec_accept(SpecState* ss, int k, const int* g, const float* logits, int V,
                        cudaGraphConditionalHandle cond, bool use_cond, cudaStream_t st) {
  launch_pdl(spec_copy_logits_kernel, dim3(2 * kNumSMs), dim3(256), 0, st, ss, k, g, logits, V);
  launch_pdl(spec_accept_kernel, dim3(1), dim3(32), 0, st, ss, k, g, cond, use_cond ? 1 : 0);
}

}  // namespace msw
