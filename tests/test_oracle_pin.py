"""Pins the CPU oracle's model arithmetic (oracle/oracle_model.c) against
implementations this repo did not write, run here on CPU:

  * transformers' LlamaForCausalLM (fp32, llama3 rope scaling) loaded with the
    oracle's own K16 fp16 weights: per-step logits of the FP16 mode, and of the
    GPTQ4 mode with the dequantised weights w = fp16((q - 8) * s);
  * the same model with every nn.Linear replaced by a torch W8A8 restatement
    (per-token absmax/127 round-half-even activations, per-channel int8
    weights, int64 matmul): INT8-mode logits;
  * vLLM's GPTQ reference quantiser (quant_utils.quantize_weights with
    scalar_types.uint4b8, group 128, vllm 0.22): its (w_q, w_s) fed through the
    oracle's W4 linear must reproduce x @ w_ref, i.e. the oracle dequantises the
    uint4b8 format exactly as vLLM defines it.

The oracle's scale rule is GPTQ's symmetric quantiser (AutoGPTQ
quant.Quantizer.find_params, sym=True: scale = 2*max|w|/15, zero = 8), which
is not vLLM's RTN test reference (scale = max(max/7, -min/8)); the two are
compared for the format, not for the scale choice.

The last test measures how much of the logit comes from the decoder layers:
ablating them moves the logits by far more than the parity bars, so the
per-step logit bars in tests/test_engine*_gpu.py test layer arithmetic.
"""
import numpy as np
import pytest

import oracle as O
from paper_2605_23057_b200.configs import model_cfg

torch = pytest.importorskip("torch")
transformers = pytest.importorskip("transformers")

SEED = 5
PROMPT = (np.arange(24, dtype=np.int32) * 131 + 7) % 2048
N_NEW = 12


def _hf_model(orc, fmt):
    """LlamaForCausalLM (fp32) holding the oracle's weights in format fmt."""
    from transformers import LlamaConfig, LlamaForCausalLM
    c = orc.cfg
    hc = LlamaConfig(vocab_size=c.vocab, hidden_size=c.hidden, intermediate_size=c.ffn,
                     num_hidden_layers=c.n_layers, num_attention_heads=c.n_heads,
                     num_key_value_heads=c.n_kv_heads, head_dim=c.head_dim,
                     rms_norm_eps=c.rms_eps, max_position_embeddings=131072,
                     rope_theta=c.rope_theta,
                     rope_scaling={"rope_type": "llama3", "factor": c.rope_factor,
                                   "low_freq_factor": c.rope_low_freq_factor,
                                   "high_freq_factor": c.rope_high_freq_factor,
                                   "original_max_position_embeddings": c.rope_orig_ctx},
                     tie_word_embeddings=False, attention_bias=False, mlp_bias=False,
                     attn_implementation="eager")
    torch.manual_seed(0)
    hf = LlamaForCausalLM(hc).float().eval()
    t = lambda a: torch.from_numpy(np.asarray(a, np.float32))

    def lin(which, layer):
        if fmt == 0:
            return t(orc.tensor(which, layer, 0))
        if fmt == 1:
            q, s = orc.tensor(which, layer, 1)
            return t(q), t(s)   # W8A8 modules take (q, s)
        q, s = orc.tensor(which, layer, fmt)
        zero = 8.0 if fmt == 2 else np.repeat(orc.tensor(which, layer, 4).astype(np.float32), 128, axis=1)
        deq = (q.astype(np.float32) - zero) * np.repeat(s.astype(np.float32), 128, axis=1)
        return t(deq.astype(np.float16))   # GPTQ4 / AWQ4 dequant rounded to fp16

    sd = {"model.embed_tokens.weight": t(orc.tensor(orc.EMBED)),
          "lm_head.weight": t(orc.tensor(orc.LM_HEAD)),
          "model.norm.weight": t(orc.tensor(orc.FINAL_NORM))}
    qd, kd = c.n_heads * c.head_dim, c.n_kv_heads * c.head_dim
    w8 = {}
    for l in range(c.n_layers):
        p = f"model.layers.{l}."
        sd[p + "input_layernorm.weight"] = t(orc.tensor(orc.ATTN_NORM, l))
        sd[p + "post_attention_layernorm.weight"] = t(orc.tensor(orc.FFN_NORM, l))
        parts = {"self_attn.o_proj": lin(orc.O, l), "mlp.gate_proj": lin(orc.GATE, l),
                 "mlp.up_proj": lin(orc.UP, l), "mlp.down_proj": lin(orc.DOWN, l)}
        qkv = lin(orc.QKV, l)
        if fmt == 1:
            (q, s) = qkv
            parts["self_attn.q_proj"] = (q[:qd], s[:qd])
            parts["self_attn.k_proj"] = (q[qd:qd + kd], s[qd:qd + kd])
            parts["self_attn.v_proj"] = (q[qd + kd:], s[qd + kd:])
        else:
            parts["self_attn.q_proj"] = qkv[:qd]
            parts["self_attn.k_proj"] = qkv[qd:qd + kd]
            parts["self_attn.v_proj"] = qkv[qd + kd:]
        for name, v in parts.items():
            if fmt == 1:
                w8[p + name] = v
                sd[p + name + ".weight"] = v[0].float()
            else:
                sd[p + name + ".weight"] = v
    missing = hf.load_state_dict(sd, strict=False)
    assert not [k for k in missing.missing_keys if "rotary" not in k], missing.missing_keys
    if fmt == 1:
        for name, (q, s) in w8.items():
            hf.get_submodule(name).forward = _w8a8_forward(q.to(torch.int64), s)
    return hf


def _w8a8_forward(q, s):
    """y = (float(sum int8 * int8 as exact integer) * s_x) * s_w, x per token."""
    def fwd(x):
        xf = x.reshape(-1, x.shape[-1]).float()
        amax = xf.abs().amax(dim=1, keepdim=True)
        sx = amax / 127.0
        xq = torch.where(amax > 0, torch.clamp(torch.round(xf / torch.where(amax > 0, sx, 1.0)),
                                               -127, 127), torch.zeros_like(xf)).to(torch.int64)
        acc = xq @ q.T   # exact int64 (|acc| < 2^31)
        y = (acc.float() * sx) * s[None, :]
        return y.reshape(*x.shape[:-1], q.shape[0])
    return fwd


@pytest.fixture(scope="module")
def orc():
    m = O.OracleModel(model_cfg("tiny"), seed=SEED, max_ctx=512, modes_mask=0xFFF)
    yield m
    m.close()


def _hf_logits(hf, prompt, toks):
    seq = np.concatenate([prompt, toks[:-1]]).astype(np.int64)
    with torch.no_grad():
        out = hf(torch.from_numpy(seq)[None]).logits[0].numpy()
    return out[len(prompt) - 1:]   # the logits that chose toks[0..n-1]


def _rel(a, b):
    return float((np.abs(a - b).max(axis=1) / b.std(axis=1)).max())


# FP16 / W4 bar: the oracle rounds every linear input and q/k/v to fp16 while
# transformers stays fp32, so the two differ by fp16 activation rounding.
# INT8: the same W8A8 arithmetic; only fp32 summation order and the fp16
# rounding of q/k/v differ (which can flip an int8 activation rounding).
@pytest.mark.parametrize("mode,fmt,tol", [(0, 0, 5e-3), (2, 2, 5e-3), (1, 1, 2e-2), (3, 3, 5e-3)])
def test_oracle_matches_transformers_llama(orc, mode, fmt, tol):
    toks, lg = orc.generate(mode, PROMPT, N_NEW, want_logits=True)
    hf = _hf_model(orc, fmt)
    ref = _hf_logits(hf, PROMPT, toks)
    assert _rel(lg, ref) < tol, f"mode {mode}: oracle vs transformers {_rel(lg, ref):.3g}"
    assert np.array_equal(ref.argmax(axis=1), toks), "greedy tokens differ from transformers"


def test_layers_carry_the_logits(orc):
    """Dropping the decoder layers (h = embedding) moves the logits by many
    times the parity bars (measured 0.39 sigma on tiny: 200x the FP16 bar of
    2e-3, 40x the INT8/W4 bar of 1e-2), so those bars test the layers."""
    toks, lg = orc.generate(0, PROMPT, N_NEW, want_logits=True)
    hf = _hf_model(orc, 0)
    hf.model.layers = torch.nn.ModuleList([])
    abl = _hf_logits(hf, PROMPT, toks)
    assert _rel(abl, lg) > 0.2, f"layer contribution only {_rel(abl, lg):.3g} sigma"


def test_oracle_w4_dequant_matches_vllm_uint4b8(orc):
    from vllm.model_executor.layers.quantization.utils.quant_utils import (
        pack_rows, quantize_weights)
    from vllm.scalar_type import scalar_types
    w = orc.tensor(orc.O, 0, 0)              # fp16 [n, k]
    n, k = w.shape
    w_ref, w_q, w_s, _ = quantize_weights(torch.from_numpy(w.T.astype(np.float32)),
                                          scalar_types.uint4b8, 128)
    q = np.ascontiguousarray(w_q.numpy().T.astype(np.uint8))      # stored uint4b8 values 0..15, [n, k]
    assert q.max() <= 15
    s = np.ascontiguousarray(w_s.numpy().T.astype(np.float16))    # [n, k/128]
    rng = np.random.default_rng(1)
    x = rng.standard_normal((3, k)).astype(np.float32)
    y = np.zeros((3, n), np.float32)
    O.lib().orc_linear(2, O._p(q), O._p(s), n, k, O._p(x), 3, O._p(y))
    x16 = x.astype(np.float16).astype(np.float32)
    # vLLM's w_ref uses the fp32 scale; the oracle stores fp16 scales and
    # rounds (q-8)*s to fp16, so build the reference from the same fp16 scale
    deq = ((q.astype(np.float32) - scalar_types.uint4b8.bias) *
           np.repeat(s.astype(np.float32), 128, axis=1)).astype(np.float16).astype(np.float32)
    ref = x16 @ deq.T
    np.testing.assert_allclose(y, ref, rtol=0, atol=2e-5 * np.abs(ref).max())
    # and with vLLM's own dequant (fp32 scales): the same up to fp16 scale rounding
    ref_v = x16 @ w_ref.numpy()
    assert np.abs(y - ref_v).max() < 5e-3 * np.abs(ref_v).max()
    # GPTQ checkpoint packing (vLLM pack_rows: qweight [k/8, n] int32, nibble i
    # of word j = row 8j+i) holds exactly the values the oracle consumes
    packed = pack_rows(w_q, 4, k, n).numpy().view(np.uint32)
    assert packed.shape == (k // 8, n)
    un = np.stack([(packed >> (4 * i)) & 0xF for i in range(8)], axis=1).reshape(k, n)
    assert np.array_equal(un.T.astype(np.uint8), q)


def test_oracle_w4_scale_rule_is_gptq_symmetric(orc):
    """orc_quant_w4_rows restates AutoGPTQ's sym Quantizer (scale 2*amax/15,
    zero 8, q = clamp(round(w/scale) + 8, 0, 15)) with the scale stored fp16."""
    w = orc.tensor(orc.GATE, 1, 0)
    q, s = orc.tensor(orc.GATE, 1, 2)
    wf = w.astype(np.float32).reshape(w.shape[0], -1, 128)
    amax = np.abs(wf).max(axis=2)
    sc = ((2.0 * amax) / 15.0).astype(np.float16)
    assert np.array_equal(sc, s)
    sf = sc.astype(np.float32)[..., None]
    qq = np.clip(np.rint(wf / np.where(sf > 0, sf, 1)) + 8, 0, 15)
    assert np.array_equal(qq.reshape(q.shape).astype(np.uint8), q)


def test_oracle_awq4_matches_autoawq_pseudo_quantize(orc):
    """orc_quant_awq4_rows restates AutoAWQ's pseudo_quantize_tensor
    (zero_point=True, w_bit=4, q_group_size=128): scales = (max - min).clamp(
    min=1e-5) / 15, zeros = (-round(min / scales)).clamp(0, 15), q = clamp(
    round(w / scales) + zeros, 0, 15), with the scale stored as fp16 first."""
    w = orc.tensor(orc.DOWN, 0, 0)
    q, s = orc.tensor(orc.DOWN, 0, 3)
    z = orc.tensor(orc.DOWN, 0, 4)
    wf = torch.from_numpy(w.astype(np.float32)).reshape(w.shape[0], -1, 128)
    mx, mn = wf.amax(dim=2, keepdim=True), wf.amin(dim=2, keepdim=True)
    sc = ((mx - mn).clamp(min=1e-5) / 15).half().float()
    zz = (-torch.round(mn / sc)).clamp(0, 15)
    qq = torch.clamp(torch.round(wf / sc) + zz, 0, 15)
    assert np.array_equal(sc.squeeze(2).half().numpy(), s)
    assert np.array_equal(zz.squeeze(2).numpy().astype(np.uint8), z)
    assert np.array_equal(qq.reshape(q.shape).numpy().astype(np.uint8), q)
    assert len(np.unique(z)) > 1  # zero points vary per group (uniform init: 7 or 8)


def test_fp8_e4m3_restatement_matches_torch():
    """oracle fp8_e4m3 (the KV-cache compression mode's rounding) equals
    torch's float8_e4m3fn conversion (round to nearest even) on every finite
    fp16 value below the saturation threshold, byte for byte."""
    import torch
    bits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    v = bits.view(np.float16)
    x = bits[np.isfinite(v) & (np.abs(v.astype(np.float32)) < 464)]
    q, y = O.fp8_e4m3(x)
    t = torch.from_numpy(x.view(np.float16).copy()).to(torch.float8_e4m3fn)
    assert np.array_equal(t.view(torch.uint8).numpy(), q)
    assert np.array_equal(t.to(torch.float16).numpy().view(np.uint16), y)
