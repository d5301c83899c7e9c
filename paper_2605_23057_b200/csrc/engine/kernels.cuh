// Launcher declarations for the sm_100a mode-executor kernels.
#pragma once

#include "common.cuh"

namespace msw {

enum WFmt { kFP16 = 0, kINT8 = 1, kW4 = 2 };

// A linear layer resident in HBM. y[n] = sum_k W[n,k] x[k].
//   kFP16: w = half [n, k] row-major
//   kINT8: w = int8 [n, k] row-major, s = float [n] per-row scale
//   kW4  : w = uint32 [n, k/8] (8 nibbles per word, interleaved so that one
//          lop3 yields the fp16 pair (k, k+1)), s = half [n, k/128]
struct LinearW {
  int fmt = kFP16;
  int n = 0, k = 0;
  const void* w = nullptr;
  const void* s = nullptr;
  const void* w_tf = nullptr;  // the same weights in tile-fragment order (decode GEMV)
  const uint8_t* z = nullptr;  // kW4 only: AWQ zero points uint8 [n, k/128] (nullptr: GPTQ, zero 8)
  size_t bytes() const {
    const size_t nk = size_t(n) * size_t(k);
    if (fmt == kFP16) return nk * 2;
    if (fmt == kINT8) return nk + size_t(n) * 4;
    return nk / 2 + size_t(n) * (k / kW4Group) * (z ? 3 : 2);
  }
};
// Engine weight slots: kFP16, kINT8, kW4 (GPTQ) and kSlotAWQ4 (a kW4 LinearW
// with zero points).
constexpr int kSlotAWQ4 = 3;
constexpr int kSlots = 4;

// ---- init.cu: K16 generator, quantisers, successor lm_head ----------------
void launch_fill_fp16(half* dst, int64_t rows, int64_t cols, uint64_t seed, uint64_t tid,
                      int scale_log2, cudaStream_t st);
void launch_fill_norm(half* dst, int64_t n, uint64_t seed, uint64_t tid, cudaStream_t st);
void launch_quant_int8(const half* w, int n, int k, int8_t* q, float* s, cudaStream_t st);
void launch_quant_w4(const half* w, int n, int k, uint32_t* packed, half* s, cudaStream_t st);
// AWQ format (AutoAWQ pseudo_quantize_tensor, zero_point=True): asymmetric
// group-128, fp16 scale (max - min) / 15, zero point, same nibble packing as W4
void launch_quant_awq4(const half* w, int n, int k, uint32_t* packed, half* s, uint8_t* z,
                       cudaStream_t st);
void launch_unpack_w4(const uint32_t* packed, int n, int k, uint8_t* nibbles, cudaStream_t st);
void launch_lm_head(const half* emb, const int* pred, const uint8_t* agree, int is_draft,
                    int V, int H, half* out, cudaStream_t st);
// out row 2i = a row i, out row 2i+1 = b row i (gate/up interleave for the SwiGLU epilogue)
void launch_interleave_rows(const void* a, const void* b, int n, size_t row_bytes, void* out,
                            cudaStream_t st);

// ---- gemv.cu: batch-1 decode GEMV ----------------------------------------
enum Prologue { kProPlain = 0, kProNorm = 1 };
enum Epilogue { kEpiStore = 0, kEpiResid = 1, kEpiSwiglu = 2, kEpiRaw = 3 };
// x: fp32 [k]. kProNorm: x <- x * rsqrt(mean(x^2)+eps) * gamma before the
// format's activation handling (fp16 rounding, or int8 absmax quantisation).
// kEpiStore: y[n] = v; kEpiResid: y[n] += v; kEpiSwiglu: y[i] = silu(v[2i]) * v[2i+1].
// kEpiRaw (INT8 only, test entry msw_linear_i8_raw): y holds the int32
// accumulators themselves, before any scale.
// x is fp32 [T, k], 1 <= T <= kGemvMaxTokens; y rows are per token.
constexpr int kGemvMaxTokens = 6;
void launch_gemv(const LinearW& W, int pro, int epi, const float* x, int T, const half* gamma,
                 float eps, float* y, cudaStream_t st,
                 const LinearW* next = nullptr);
void launch_gemv_i8_acc(const int8_t* w, const int8_t* x, int n, int k, int* acc, cudaStream_t st);
// row-major weights (FP16 half / INT8 int8 / W4 row-packed words) -> the
// tile-fragment layout the decode GEMV streams (same byte count)
size_t tf_bytes(int fmt, int n, int k);
void launch_repack_tf(int fmt, const void* src, int n, int k, void* dst, cudaStream_t st);

// ---- gemm.cu: T > 1 tokens (prefill / verify / continuous batching) -----------
// prep: per token row, optional RMSNorm, then fp16 rounding (xh) or int8
// quantisation (xq + per-token scale).
void launch_prep_act(int fmt, const float* x, int T, int K, const half* gamma, float eps,
                     half* xh, int8_t* xq, float* xscale, cudaStream_t st);
void launch_gemm(const LinearW& W, int epi, const half* xh, const int8_t* xq, const float* xscale,
                 int T, float* y, cudaStream_t st);

// ---- gemm_tc.cu: tcgen05/TMEM/TMA tensor-core path (n % 128 == 0, k % 128 == 0)
bool gemm_tc_supported(const LinearW& W);
void launch_gemm_tc(const LinearW& W, int epi, const half* xh, const int8_t* xq,
                    const float* xscale, int T, float* y, cudaStream_t st);

// ---- attention.cu -----------------------------------------------------------
struct AttnShape {
  int n_heads, n_kv_heads, head_dim;
  int max_blocks_per_seq;  // block-table row stride
  int n_blocks = 0;        // KV pool blocks per layer (tensor maps over the pool)
};
// qkv fp32 [T, (Hq+2Hk)*D] -> RoPE on q,k -> q fp16 [T,Hq,D]; k,v fp16 into the
// paged cache at slot[t] (= block*16 + offset) of this layer.
// RoPE cos/sin table [max_pos][head_dim/2] (fp32 angle pos * inv_freq, as the oracle)
void launch_rope_table(const float* inv_freq, int head_dim, int max_pos, float2* table,
                       cudaStream_t st);
void launch_rope_append(const float* qkv, int T, const int* pos, const int* slot,
                        const float2* rope, const AttnShape& a, half* q_out, half* kc, half* vc,
                        cudaStream_t st);
// o fp32 [T, Hq, D]: token t (sequence seq_of[t], position pos[t]) attends to
// positions [0, pos[t]] of its sequence through block_table[seq_of[t]].
void launch_attention(const half* q, int T, const int* pos, const int* seq_of,
                      const int* block_table, const half* kc, const half* vc, const AttnShape& a,
                      int nsplit, float* part_o, float* part_ml, float* o, cudaStream_t st);

// Same semantics on the tensor pipe (attn_prefill.cu): many query tokens,
// packed from any number of sequences; no split-KV (o written directly).
// head_dim 128 runs on tcgen05 (attn_prefill_tc05.cu, TMA + TMEM); needs
// a.n_blocks (the KV pool is addressed through TMA tensor maps).
bool attention_prefill_tc05_supported(const AttnShape& a);
void launch_attention_prefill_tc05(const half* q, int T, const int* pos, const int* seq_of,
                                   const int* block_table, const half* kc, const half* vc,
                                   uint64_t kv_rows, const AttnShape& a, float* o, cudaStream_t st);
void launch_attention_prefill(const half* q, int T, const int* pos, const int* seq_of,
                              const int* block_table, const half* kc, const half* vc,
                              const AttnShape& a, float* o, cudaStream_t st);

// Decode / continuous batching (each token is the newest of its own sequence):
// RoPE + KV append fused into the attention kernel; reads fp32 qkv directly.
// run = true: the T <= 6 tokens are consecutive positions of ONE sequence
// (speculative verify, the draft's catch-up step, short prefills); token t's
// CTAs take the keys / values of tokens 0..t from the qkv rows instead of the
// cache, so no separate RoPE/append launch is needed.
void launch_attention_decode(const float* qkv, const float2* rope, int T, const int* pos,
                             const int* slot, const int* seq_of, const int* block_table, half* kc,
                             half* vc, const AttnShape& a, int nsplit, float* part_o,
                             float* part_ml, int* counters, float* o, cudaStream_t st,
                             bool run = false);
// KV-cache compression mode: the same kernel on an FP8 E4M3 paged cache
// (history widened while staged; new keys / values rounded through E4M3).
void launch_attention_decode_kv8(const float* qkv, const float2* rope, int T, const int* pos,
                                 const int* slot, const int* seq_of, const int* block_table,
                                 uint8_t* kc, uint8_t* vc, const AttnShape& a, int nsplit,
                                 float* part_o, float* part_ml, int* counters, float* o,
                                 cudaStream_t st, bool run = false);
// positions [0, npos) of one sequence, every layer: fp16 cache (blocks b16)
// -> E4M3 cache (blocks b8); b16 / b8 are device block lists
void launch_kv_compress(const half* kc, const half* vc, uint8_t* kc8, uint8_t* vc8,
                        size_t layer_elems, int layers, const int* b16, const int* b8, int npos,
                        int Hk, int D, cudaStream_t st);
// test entry: q = E4M3(x) (RNE, satfinite), y = fp16(q); n even
void launch_fp8_roundtrip(const half* x, int64_t n, uint8_t* q, half* y, cudaStream_t st);

// ---- misc.cu ------------------------------------------------------------------
void launch_embed(const half* emb, const int* tok, int T, int H, float* h, cudaStream_t st);
// out[t] = argmax_v logits[t, v] (lowest index on ties)
// ws: 2*T zeroed u64 words (slots + counters), left zeroed on return.
void launch_argmax(const float* logits, int T, int V, int* out, unsigned long long* ws,
                   cudaStream_t st);
void launch_gather_rows(const float* src, const int* rows, int n, int width, float* dst,
                        cudaStream_t st);
// batch-1 decode bookkeeping for graph replay: tok = history[step] = next[0],
// step += 1, pos += 1, slot from block-table row 0
void launch_advance(const int* next, int* tok, int* pos, int* slot, int* step, int* history,
                    const int* block_table, cudaStream_t st);
// continuous batching: hist[hbase[t] + pos[t]] = tok[t] = next[t]; pos[t] += 1;
// slot[t] from block-table row seq_of[t]
void launch_cb_advance(const int* next, int T, int* tok, int* pos, int* slot, const int* seq_of,
                       const int* hbase, int* hist, const int* block_table, int bt_stride,
                       cudaStream_t st);

// ---- speculative decoding state (device) and round kernels (misc.cu) ----------
constexpr int kSpecMaxK = 8;
struct SpecState {
  int n;         // committed sequence length (prompt + emitted)
  int emitted;   // tokens emitted so far
  int n_new;     // tokens to emit
  int rounds, proposed, accepted;
  int last;      // seq[n-1]
  int prev;      // seq[n-2]
  int props[kSpecMaxK];  // this round's draft proposals
  int* out;             // emitted tokens [n_new]
  float* logits_out;    // optional [n_new, V] logits of the emitted tokens
};
void launch_spec_init(SpecState* ss, const int* next, int plen, int n_new, int prompt_last,
                      float* logits_out, cudaStream_t st);
void launch_spec_draft_setup(const SpecState* ss, int* tok, int* pos, int* slot, int* seq_of,
                             int* logit_rows, const int* block_table, cudaStream_t st);
void launch_spec_draft_next(SpecState* ss, int i, const int* next, int* tok, int* pos, int* slot,
                            int* seq_of, const int* block_table, cudaStream_t st);
void launch_spec_verify_setup(SpecState* ss, int k, const int* next, int* tok, int* pos, int* slot,
                              int* seq_of, const int* block_table, cudaStream_t st);
// two launches (logits copy, accept); use_cond: accept sets the enclosing WHILE node's condition
void launch_spec_accept(SpecState* ss, int k, const int* g, const float* logits, int V,
                        cudaGraphConditionalHandle cond, bool use_cond, cudaStream_t st);

}  // namespace msw
