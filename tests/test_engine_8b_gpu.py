"""Production-shape parity on the B200: the Llama-3.1-8B-shape engine (the
shapes the bench runs: K = 4096 / 14336 decode GEMVs, 32 q / 8 kv heads of
128, vocab 128256) against the CPU oracle on the same K16 weights, batch-1,
in FP16, INT8 and GPTQ4 (and GPTQ + prefix caching on a repeated prompt).

This is the only test that drives the 8B-specialised decode kernels (the W4
issue-lean GEMV with register-resident activation fragments, the 8B attention
splits) through their fused RMSNorm / SwiGLU / residual epilogues. Bars as in
test_engine_gpu: tokens bit-exact, logits within the per-mode tolerance."""
import numpy as np
import pytest

import oracle as O
from paper_2605_23057_b200 import (MODE_FP16, MODE_GPTQ4, MODE_GPTQ_PC, MODE_INT8, engine_cfg,
                                   model_cfg)
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
TOL = {MODE_FP16: 2e-3, MODE_INT8: 5e-2, MODE_GPTQ4: 1e-2, MODE_GPTQ_PC: 1e-2}
ORACLE_MODE = {MODE_FP16: 0, MODE_INT8: 1, MODE_GPTQ4: 2, MODE_GPTQ_PC: 2}


@pytest.fixture(scope="module")
def pair8b(cuda_ok):
    modes = (MODE_FP16, MODE_INT8, MODE_GPTQ4, MODE_GPTQ_PC)
    eng = Engine(engine_cfg(target="llama8b", draft=None, modes=modes, seed=3, kv_blocks=96,
                            max_seq_len=512))
    orc = O.OracleModel(model_cfg("llama8b"), seed=3, max_ctx=512, modes_mask=0b111)
    yield eng, orc
    eng.close()
    orc.close()


@pytest.mark.parametrize("mode", [MODE_FP16, MODE_INT8, MODE_GPTQ4])
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
