"""Production-shape parity on the B200: the Llama-3.1-8B-shape engine (the
shapes the bench runs: K = 4096 / 14336 decode GEMVs, 32 q / 8 kv heads of
128, vocab 128256) against the CPU oracle on the same K16 weights, batch-1,
in FP16, INT8, GPTQ4, AWQ4 and KV-cache compression (and GPTQ + prefix caching on a repeated prompt).

This is the only test that drives the 8B-specialised decode kernels (the W4
issue-lean GEMV with register-resident activation fragments, the 8B attention
splits) through their fused RMSNorm / SwiGLU / residual epilogues. Bars as in
test_engine_gpu: tokens bit-exact, logits within the per-mode tolerance."""
import numpy as np
import pytest

import oracle as O
from paper_2605_23057_b200 import (MODE_AWQ4, MODE_FP16, MODE_KV_COMPRESSION, MODE_GPTQ4, MODE_GPTQ_PC, MODE_INT8, MODE_INT8_CB,
                                   MODE_SPEC, engine_cfg, model_cfg)
from paper_2605_23057_b200.engine import Engine

pytestmark = pytest.mark.gpu

# INT8 (W8A8, per-token dynamic activation quantisation) is discontinuous: a
# 1-ulp fp32 difference (GPU vs oracle summation order in RMSNorm, attention or
# the tcgen05 prefill) eventually flips one int8 rounding; that perturbs the
# next layer by a full quantum, which flips many more, and over 32 layers the
# two trajectories separate to the quantisation-noise level itself (measured:
# GPU-vs-oracle 3.1 % of the logit std, oracle INT8-vs-FP16 3.6 %). Tokens stay
# exact. The bar: < 5e-2, and no larger than 1.5x the oracle's own INT8-vs-FP16
# error on the same prompt. The int32 accumulations themselves are bit-exact
# (test_kernels_gpu).
TOL = {MODE_FP16: 2e-3, MODE_INT8: 5e-2, MODE_GPTQ4: 1e-2, MODE_AWQ4: 1e-2, MODE_GPTQ_PC: 1e-2,
       MODE_KV_COMPRESSION: 1e-2}
ORACLE_MODE = {MODE_FP16: 0, MODE_INT8: 1, MODE_GPTQ4: 2, MODE_AWQ4: 3, MODE_GPTQ_PC: 2, MODE_KV_COMPRESSION: 9}


@pytest.fixture(scope="module")
def pair8b(cuda_ok):
    modes = (MODE_FP16, MODE_INT8, MODE_GPTQ4, MODE_AWQ4, MODE_GPTQ_PC, MODE_SPEC, MODE_INT8_CB,
             MODE_KV_COMPRESSION)
    eng = Engine(engine_cfg(target="llama8b", draft="llama1b", modes=modes, seed=3, kv_blocks=256,
                            max_batch=64, max_seq_len=512))
    orc = O.OracleModel(model_cfg("llama8b"), seed=3, max_ctx=512, modes_mask=0b1111)
    yield eng, orc
    eng.close()
    orc.close()


@pytest.mark.parametrize("mode", [MODE_FP16, MODE_INT8, MODE_GPTQ4, MODE_AWQ4, MODE_KV_COMPRESSION])
def test_8b_batch1_decode_matches_oracle(pair8b, mode):
    eng, orc = pair8b
    p = (np.random.default_rng(40 + mode).integers(0, eng.vocab, size=21)).astype(np.int32)
    r = eng.run(mode, p, 4, want_logits=True)
    toks, lg = orc.generate(ORACLE_MODE[mode], p, 4, want_logits=True)
    assert np.array_equal(r.tokens, toks)
    err = np.abs(r.logits - lg).max(axis=1) / lg.std(axis=1)
    assert err.max() < TOL[mode], f"logit error {err.max():.3g}"
    if mode == MODE_INT8:
        _, lg16 = orc.generate(0, p, 4, want_logits=True)
        qerr = np.abs(lg16 - lg).max(axis=1) / lg.std(axis=1)
        assert (err < 1.5 * qerr).all(), f"flip noise {err} vs quantisation error {qerr}"
        # the INT8 mode really runs W8A8: its distance from the FP16 oracle is the
        # quantisation error, an order of magnitude above the FP16 mode's bar (an
        # engine that silently ran FP16 weights here would sit within TOL[FP16])
        e16 = np.abs(r.logits - lg16).max(axis=1) / lg16.std(axis=1)
        assert (e16 > 5 * TOL[MODE_FP16]).all(), f"INT8 mode within FP16 tolerance of FP16: {e16}"


def test_8b_graph_decode_and_prefix_reuse(pair8b):
    eng, orc = pair8b
    p = (np.random.default_rng(7).integers(0, eng.vocab, size=40)).astype(np.int32)
    ref, _ = orc.generate(2, p, 12)
    r = eng.run(MODE_GPTQ4, p, 12)  # CUDA-graph decode loop
    assert np.array_equal(r.tokens, ref)
    eng.run(MODE_GPTQ_PC, p, 12)
    r2 = eng.run(MODE_GPTQ_PC, p, 12)  # the 2 full prompt blocks now come from the prefix cache
    assert r2.prefix_hit_tokens == 32
    assert np.array_equal(r2.tokens, ref)


def test_8b_continuous_batching_ragged_64(pair8b):
    """BASELINE config 3b's shape: a ragged cohort of 64 co-scheduled INT8
    requests at 8B (tcgen05 kind::i8 GEMMs with the deterministic split-K for
    T > 6 live rows, CUDA-graph steps between retirements). Every sequence's
    tokens equal the GPU batch-1 INT8 mode's; a spread of 6 sequences is
    checked against the oracle (tokens exact, logits within the INT8 bar)
    every step; a repeated cohort is bitwise identical."""
    eng, orc = pair8b
    rng = np.random.default_rng(64)
    plens = [int(x) for x in rng.integers(1, 8, size=64)]
    nnew = [int(x) for x in rng.integers(2, 6, size=64)]
    prompts = [rng.integers(0, eng.vocab, size=n).astype(np.int32) for n in plens]
    res = eng.run_batch(MODE_INT8_CB, prompts, nnew, want_logits=True)
    again = eng.run_batch(MODE_INT8_CB, prompts, nnew, want_logits=True)
    for i in range(64):
        assert np.array_equal(res[i].tokens, again[i].tokens), i
        assert np.array_equal(res[i].logits.view(np.uint32), again[i].logits.view(np.uint32)), i
        single = eng.run(MODE_INT8, prompts[i], nnew[i])
        assert np.array_equal(res[i].tokens, single.tokens), i
    for i in (0, 13, 31, 32, 50, 63):
        toks, lg = orc.generate(1, prompts[i], nnew[i], want_logits=True)
        assert np.array_equal(res[i].tokens, toks), i
        err = np.abs(res[i].logits - lg).max(axis=1) / lg.std(axis=1)
        assert err.max() < TOL[MODE_INT8], f"request {i}: logit error {err.max():.3g}"


def test_8b_speculative_1b_draft(pair8b):
    """BASELINE config 4's pair: the 1B-shape FP16 draft proposes k = 4
    tokens per round for the 8B-shape FP16 target (device-resident rounds in
    one WHILE-node graph). 64 tokens equal the target's greedy tokens; round,
    proposal and accept counts equal the oracle's; logits of every emitted
    token within the FP16 bar."""
    eng, orc = pair8b
    drf = O.OracleModel(model_cfg("llama1b"), seed=3, is_draft=True, max_ctx=512)
    p = np.random.default_rng(5).integers(0, eng.vocab, size=6).astype(np.int32)
    r = eng.run(MODE_SPEC, p, 64, want_logits=True)
    toks, lg, st = O.spec_generate(orc, drf, 4, p, 64, want_logits=True)
    drf.close()
    assert np.array_equal(r.tokens, toks)
    assert (r.spec_rounds, r.spec_proposed, r.spec_accepted) == (st["rounds"], st["proposed"], st["accepted"])
    assert 0 < r.spec_accepted < r.spec_proposed
    err = np.abs(r.logits - lg).max(axis=1) / lg.std(axis=1)
    assert err.max() < TOL[MODE_FP16], f"logit error {err.max():.3g}"
    g = eng.run(MODE_SPEC, p, 64)  # graph path (no logits)
    assert np.array_equal(g.tokens, toks) and g.spec_rounds == st["rounds"]
