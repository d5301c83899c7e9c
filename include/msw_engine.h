/* modeswitch-b200: C ABI of the per-GPU mode executor (libmsw_engine.so).
 *
 * This is the layer the reference's simulator seam hands off to: the
 * reference computes a routed mode's latency as
 *     fp16_latency / cell.latency_speedup + overhead     (sim.cpp:132-135)
 * inside simulate_request (sim.hpp:92-96, sim.cpp:80-145). Here the routed
 * mode is executed on a B200 instead and the measured latency/tokens come
 * back through msw_result. Routing (RulePolicy::route) stays host C++ in
 * libmodeswitch.so; modes are the reference's InferenceMode integers
 * (domain.hpp:71-84).
 *
 * Entry points and the reference interface each replaces:
 *   msw_engine_create    <- default_profile()/load_profile() (profile.cpp:132-239, 312-450):
 *                           instead of loading measured ratios, materialise
 *                           every routable mode's weights resident in HBM.
 *   msw_engine_run       <- simulate_request() for batch-1 modes
 *                           (FP16, INT8, GPTQ4, SpeculativeDecoding, GPTQPlusPrefixCaching)
 *   msw_engine_run_batch <- simulate_request() for INT8PlusContinuousBatching
 *                           (a co-scheduled cohort, batching guard sim.cpp:104-106)
 *   msw_last_error       <- the DataError/ConfigError message (domain.hpp:12-27)
 *   msw_engine_destroy   <- (no reference counterpart; engine owns device memory)
 *
 * Return codes: 0 ok; 2 config (bad mode id, shapes, mode not resident);
 * 3 data (bad token ids / lengths; caller applies the FP16 fallback as
 * sim.cpp:112-124 does); 1 CUDA/other. No C++ exception crosses the ABI.
 * One engine per device, driven by one host thread at a time.
 */
#ifndef MSW_ENGINE_H_
#define MSW_ENGINE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* InferenceMode integer values (reference domain.hpp:71-84). */
enum {
  MSW_MODE_FP16 = 0,
  MSW_MODE_INT8 = 1,
  MSW_MODE_GPTQ4 = 2,
  MSW_MODE_AWQ4 = 3,            /* AWQ-format W4: asymmetric g128 (scale + zero point) (screening mode) */
  MSW_MODE_SPECULATIVE = 4,
  MSW_MODE_CHUNKED_PREFILL = 6, /* FP16, prefill in 512-token chunks (screening mode) */
  MSW_MODE_CUDA_GRAPHS = 8,     /* FP16, graph-replayed decode (screening mode) */
  MSW_MODE_KV_COMPRESSION = 9,  /* FP16 weights, FP8 E4M3 KV cache after prefill (screening mode) */
  MSW_MODE_GPTQ_PREFIX_CACHING = 10,
  MSW_MODE_INT8_CONT_BATCHING = 11
};

/* Weight formats of a linear layer. */
enum { MSW_W_FP16 = 0, MSW_W_INT8 = 1, MSW_W_W4G128 = 2, MSW_W_AWQ4 = 3 };

#define MSW_KV_BLOCK 16 /* tokens per paged-KV block */
#define MSW_W4_GROUP 128

/* Llama-architecture shape. All K dims must be multiples of 128. */
typedef struct msw_model_cfg {
  int32_t hidden;
  int32_t n_layers;
  int32_t n_heads;
  int32_t n_kv_heads;
  int32_t head_dim; /* 64 or 128 */
  int32_t ffn;
  int32_t vocab;
  float rms_eps;    /* 1e-5 */
  float rope_theta; /* 500000 */
  /* llama3 rope scaling; rope_factor <= 0 disables it */
  float rope_factor;           /* 8 */
  float rope_low_freq_factor;  /* 1 */
  float rope_high_freq_factor; /* 4 */
  int32_t rope_orig_ctx;       /* 8192 */
} msw_model_cfg;

typedef struct msw_engine_cfg {
  msw_model_cfg target;
  msw_model_cfg draft;  /* used when has_draft */
  int32_t has_draft;
  uint32_t modes_mask;  /* bit (1u << InferenceMode) for each resident mode */
  uint64_t weight_seed; /* K16 deterministic init; identical on the CPU oracle */
  int32_t draft_agree_permille; /* vocab fraction where draft successor == target's */
  int32_t kv_blocks;     /* paged KV pool size in blocks (per model) */
  int32_t max_batch;     /* live sequences in one continuous-batching step (<= 64) */
  int32_t max_seq_len;   /* per sequence, tokens (prompt + generated + spec slack) */
  int32_t spec_k;        /* draft proposals per round (4) */
  int32_t use_graphs;    /* capture the decode step in a CUDA graph */
} msw_engine_cfg;

typedef struct msw_request {
  int32_t mode;              /* InferenceMode value */
  const int32_t* prompt_ids; /* HOST pointer, prompt_len token ids */
  int32_t prompt_len;
  int32_t max_new_tokens;    /* tokens to generate (>= 1) */
  int32_t prefix_group;      /* informational; prefix reuse is content-hashed */
  int32_t prefix_len;
  uint64_t seq;              /* caller's sequence number */
} msw_request;

typedef struct msw_result {
  int32_t* out_ids;     /* HOST buffer, capacity max_new_tokens */
  int32_t n_out;
  float* logits;        /* optional HOST buffer [max_new_tokens, vocab] or NULL */
  double prefill_ms;    /* device time, CUDA events */
  double decode_ms;
  double total_ms;      /* admission to last token, incl. host<->device copies */
  int32_t spec_rounds;
  int32_t spec_proposed;
  int32_t spec_accepted;
  int32_t prefix_hit_tokens;
  int32_t kernel_launches; /* engine kernels launched for this request */
} msw_result;

typedef struct msw_engine msw_engine;

int msw_engine_create(int device, const msw_engine_cfg* cfg, msw_engine** out);
int msw_engine_run(msw_engine* e, const msw_request* req, msw_result* res);
int msw_engine_run_batch(msw_engine* e, const msw_request* reqs, int32_t n,
                         msw_result* res);
void msw_engine_destroy(msw_engine* e);
const char* msw_last_error(void);

/* Resident HBM bytes per mode's weights (all linears + lm_head), the
 * algorithmic bytes one batch-1 decode token streams. */
int msw_engine_weight_bytes(msw_engine* e, int32_t mode, int64_t* bytes);
/* HBM footprint of serving one request of `tokens` positions in `mode`: the
 * mode's resident weights (speculative decoding: target FP16 + draft) plus
 * the request's K/V cache (target, and draft for speculative decoding). The
 * executor's memory_ratio (reference SimRequestResult::memory_ratio,
 * sim.hpp:49) is this over the FP16 figure for the same request. */
int msw_engine_memory_bytes(msw_engine* e, int32_t mode, int32_t tokens, int64_t* bytes);
/* Drops every cached prefix block (prefix caching) and resets counters. */
int msw_engine_reset_prefix_cache(msw_engine* e);

/* KV-cache compression mode test entry: q[i] = FP8 E4M3 of the fp16 x[i]
 * (round to nearest even, saturating to +-448), y[i] = q[i] widened back to
 * fp16 (exact). n even; device pointers. */
int msw_fp8_e4m3_roundtrip(const uint16_t* x, int64_t n, uint8_t* q, uint16_t* y, void* stream);

/* ---- kernel-level entry points (device pointers; used by parity tests and
 * bench.py to time the dominant kernel). stream may be NULL (legacy). ---- */

/* y[T,N] = x[T,K] . W^T for one weight format. x is fp32 [T,K]; y fp32.
 * INT8: x is quantised per token inside the kernel (absmax/127, RNE).
 * W4: w = (q-8)*s_g, q row-packed (word j = k 8j..8j+7, nibble position
 * (i>>1) + 4*(i&1) for element i). */
int msw_linear(int32_t wtype, const void* w, const void* scales, int32_t n,
               int32_t k, const float* x, int32_t t, float* y, void* stream);

/* Decode GEMV (t <= 6 tokens) on weights already in the engine's decode
 * (tile-fragment) layout, see msw_repack_decode. */
int msw_linear_decode(int32_t wtype, const void* w_tf, const void* scales, int32_t n, int32_t k,
                      const float* x, int32_t t, float* y, void* stream);
/* Row-major weights (fp16 / int8 / W4 row-packed) -> the decode layout:
 * 16-row tiles of 512-byte mma.sync A-fragment chunks; same byte count. */
int msw_repack_decode(int32_t wtype, const void* w, int32_t n, int32_t k, void* out, void* stream);

/* The W8A8 PRODUCTION kernels' raw int32 accumulators: w int8 [n,k]
 * row-major, x fp32 [t,k] quantised per token exactly as in the engine
 * (absmax/127, RNE), acc int32 [t,n] = sum_k w[n,k] * q(x)[t,k] before any
 * scale. t <= 6 runs the decode GEMV (gemv_tf_kernel<INT8>, mma.sync s8),
 * t > 6 the tcgen05 kind::i8 GEMM including its split-K combine. With
 * integer x and max|x[t]| = 127 the quantisation is the identity. */
int msw_linear_i8_raw(const int8_t* w, int32_t n, int32_t k, const float* x, int32_t t,
                      int32_t* acc, void* stream);

/* INT8 core on identical operands: acc[n] = sum_k w[n,k]*x[k] (int32 exact). */
int msw_gemv_i8_acc(const int8_t* w, const int8_t* x, int32_t n, int32_t k,
                    int32_t* acc, void* stream);

/* K16 generator: fills a fp16 [rows, cols] tensor of the given tensor id the
 * way the engine initialises weights (uniform * 2^-scale_log2). */
int msw_fill_fp16(uint16_t* dst, int64_t rows, int64_t cols, uint64_t seed,
                  uint64_t tensor_id, int32_t scale_log2, void* stream);

/* Quantisers used at engine init, exposed for parity tests. */
int msw_quant_int8_rows(const uint16_t* w, int32_t n, int32_t k, int8_t* q,
                        float* scales, void* stream);
/* AWQ4 (AWQ format: asymmetric group-128, y = sum_g s_g sum (q - z_g) x):
 * w row-packed words [n][k/8] as W4, fp16 scales and uint8 zero points
 * [n][k/128]; same dispatch as msw_linear (decode GEMV t <= 6, tcgen05 GEMM). */
int msw_linear_awq4(const void* w, const void* scales, const uint8_t* zeros, int32_t n, int32_t k,
                    const float* x, int32_t t, float* y, void* stream);
/* AWQ4 quantiser (AutoAWQ pseudo_quantize_tensor, zero_point=True), bit-identical
 * to oracle/orc_quant_awq4_rows (packing as msw_quant_w4_rows). */
int msw_quant_awq4_rows(const uint16_t* w, int32_t n, int32_t k, uint8_t* packed, uint16_t* scales,
                        uint8_t* zeros, void* stream);
int msw_quant_w4_rows(const uint16_t* w, int32_t n, int32_t k, uint8_t* packed,
                      uint16_t* scales, void* stream);

/* Decode / continuous-batching attention (attn_decode_kernel, the engine's
 * kernel): T query tokens, each the newest token of its own sequence.
 * qkv fp32 [T, (Hq+2Hk)*D] (pre-RoPE); rope float2 [max_pos][D/2] (cos, sin);
 * pos / slot / seq_of int32 [T]; block_table int32 [rows, max_blocks];
 * kc / vc fp16 paged cache [nblk][Hk][16][D] (one layer). RoPE is applied to
 * q and the new k, k / v are appended at slot[t], and o fp32 [T, Hq, D] is
 * softmax(q k^T / sqrt(D)) v over positions [0, pos[t]], split over nsplit
 * CTAs per (token, kv head) and merged in-kernel. */
int msw_attention_decode(const float* qkv, const void* rope, int32_t T, const int32_t* pos,
                         const int32_t* slot, const int32_t* seq_of, const int32_t* block_table,
                         int32_t max_blocks, uint16_t* kc, uint16_t* vc, int32_t n_heads,
                         int32_t n_kv_heads, int32_t head_dim, int32_t nsplit, float* o,
                         void* stream);

int msw_device_sync(void);

/* PCI bus id ("0000:1b:00.0") of CUDA device `device`, for resolving the
 * matching NVML handle (energy sampling) independent of CUDA_VISIBLE_DEVICES. */
int msw_device_pci_bus_id(int32_t device, char* buf, int32_t len);

#ifdef __cplusplus
}
#endif

#endif /* MSW_ENGINE_H_ */
