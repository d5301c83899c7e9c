/* CPU ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the mode executor's arithmetic, used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * as the checker. It is never linked into, or called by, the product path
 * (paper_2605_23057_b200/lib/ shared objects).
 *
 * Parity status: the reference (/root/reference) contains no inference
 * arithmetic (SPEC.md:20 puts "actual GPU inference" out of scope), so no
 * reference golden vector pins a logit or token; the reference pins only the
 * routing side, checked against oracle/_ref. The model math is pinned
 * instead against implementations run in this container
 * (tests/test_oracle_pin.py): transformers 5.5 LlamaForCausalLM (fp32) with
 * this oracle's weights matches the FP16, GPTQ4 and INT8 (torch W8A8
 * restatement) logits within 7.5e-4 / 7.0e-4 / 3.5e-3 of the logit std, with
 * identical greedy tokens; vLLM 0.22 quant_utils' uint4b8 (w_q, w_s) run
 * through the W4 linear reproduces the dequantised product. Its building
 * blocks follow public definitions:
 *   - Llama-3 decoder forward, llama3 RoPE scaling per transformers
 *     modeling_rope_utils.py:_compute_llama3_parameters (theta 500000,
 *     factor 8, low 1, high 4, original 8192);
 *   - GPTQ symmetric uint4b8 group-128 dequant w = (q - 8) * s (vLLM
 *     quant_utils.py pack/quantize conventions), RTN quantisation;
 *   - W8A8: per-output-channel int8 weights, per-token absmax/127 dynamic
 *     activation quantisation, round-half-even, int32 accumulation;
 *   - greedy argmax, lowest index wins ties; speculative decoding emits the
 *     target's greedy tokens.
 */
#ifndef MSW_ORACLE_MODEL_H_
#define MSW_ORACLE_MODEL_H_

#include <stdint.h>

#include "../include/msw_engine.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_model orc_model;

/* is_draft selects the draft tensor-id space and successor map. */
orc_model* orc_model_create(const msw_model_cfg* cfg, uint64_t seed,
                            int is_draft, int32_t draft_agree_permille,
                            uint32_t modes_mask, int32_t max_ctx);
void orc_model_destroy(orc_model* m);

/* Greedy generation in one mode (FP16=0, INT8=1, GPTQ4=2, AWQ4=3). logits optional
 * [n_new, vocab]. Returns 0 on success. */
int orc_generate(orc_model* m, int mode, const int32_t* prompt, int plen,
                 int n_new, int32_t* out, float* logits);

/* Speculative decoding: draft proposes k greedy tokens, target verifies. The
 * emitted tokens equal the target's greedy tokens; proposed/accepted counts
 * are deterministic given the tokens. target_mode is FP16. */
int orc_spec_generate(orc_model* target, orc_model* draft, int k,
                      const int32_t* prompt, int plen, int n_new, int32_t* out,
                      float* logits, int32_t* rounds, int32_t* proposed,
                      int32_t* accepted);

/* Successor map of the peaked init: next token the model predicts for t. */
int32_t orc_successor(orc_model* m, int32_t t);

/* Building blocks, for kernel-level parity tests. */
void orc_fill_fp16(uint16_t* dst, int64_t rows, int64_t cols, uint64_t seed,
                   uint64_t tensor_id, int32_t scale_log2);
void orc_quant_int8_rows(const uint16_t* w, int32_t n, int32_t k, int8_t* q,
                         float* scales);
/* q_out: one nibble value (0..15) per byte, [n, k]; scales fp16 [n, k/128] */
void orc_quant_w4_rows(const uint16_t* w, int32_t n, int32_t k, uint8_t* q_out,
                       uint16_t* scales);
/* AWQ format, asymmetric group-128: q nibble-per-byte [n, k], fp16 scales and
 * uint8 zero points [n, k/128]; w' = (q - z) * s. */
/* KV-cache compression: FP8 E4M3 (RNE, saturating) of fp16 values: q the
 * E4M3 byte, y its fp16 value. */
void orc_fp8_e4m3_roundtrip(const uint16_t* x, int64_t n, uint8_t* q, uint16_t* y);
void orc_quant_awq4_rows(const uint16_t* w, int32_t n, int32_t k, uint8_t* q_out,
                         uint16_t* scales, uint8_t* zeros);
void orc_linear_awq4(const uint8_t* q, const uint16_t* scales, const uint8_t* zeros, int32_t n,
                     int32_t k, const float* x, int32_t t, float* y);
void orc_gemv_i8_acc(const int8_t* w, const int8_t* x, int32_t n, int32_t k,
                     int32_t* acc);
/* y[t,n] = sum_k W[n,k] x[t,k] with the mode's activation handling. */
void orc_linear(int wtype, const void* w, const void* scales, int32_t n,
                int32_t k, const float* x, int32_t t, float* y);
int orc_threads(void);

/* Copy one of the model's tensors out (for pinning this restatement against
 * independent implementations, e.g. transformers' LlamaForCausalLM).
 * which: 0 embed [V,h] fp16, 1 lm_head [V,h] fp16, 2 final_norm [h] fp16,
 *        3 attn_norm [h], 4 ffn_norm [h] (layer l),
 *        5 qkv, 6 o, 7 gate, 8 up, 9 down (layer l, format fmt):
 *          fmt 0: w fp16 [n,k];   fmt 1: w int8 [n,k], s fp32 [n];
 *          fmt 2 (GPTQ4) / 3 (AWQ4): w nibble-per-byte [n,k], s fp16 [n,k/128];
 *          fmt 4: the AWQ4 zero points uint8 [n,k/128] into w.
 * Returns 0, or -1 if the tensor/format is not resident. */
int orc_model_tensor(orc_model* m, int which, int layer, int fmt, void* w, void* s);

#ifdef __cplusplus
}
#endif
#endif
