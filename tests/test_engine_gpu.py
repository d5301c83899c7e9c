"""End-to-end mode parity on the B200 through the C ABI (msw_engine_run /
msw_engine_run_batch) against the CPU oracle on the same K16 random-init
weights and synthetic prompts.

Bars:
  * greedy tokens bit-exact in every mode (FP16, INT8, GPTQ4, AWQ4, spec, GPTQ+PC, INT8+CB);
  * speculative decoding: tokens == target greedy, and round/proposal/accept
    counts equal the oracle's (they are a deterministic function of tokens);
  * logits: max |gpu - oracle| / std(oracle logits) < 2e-3 (FP16),
    < 1e-2 (W4 GPTQ / AWQ: fp16 partial sums) — per generated step. INT8: < 1e-2 (a 1-ulp
    difference in an fp32 activation can flip one int8 activation rounding, and
    the tensor-core prefill attention rounds P to fp16; tokens stay exact).
"""
import numpy as np
import pytest

import oracle as O
from paper_2605_23057_b200 import (MODE_AWQ4, MODE_CHUNKED_PREFILL, MODE_CUDA_GRAPHS, MODE_KV_COMPRESSION, MODE_FP16, MODE_GPTQ4,
                                   MODE_GPTQ_PC, MODE_INT8, MODE_INT8_CB, MODE_SPEC, engine_cfg,
                                   model_cfg)
from paper_2605_23057_b200._capi import MswError
from paper_2605_23057_b200.engine import Engine

pytestmark = pytest.mark.gpu

TOL = {MODE_FP16: 2e-3, MODE_INT8: 1e-2, MODE_GPTQ4: 1e-2, MODE_AWQ4: 1e-2, MODE_KV_COMPRESSION: 1e-2, MODE_GPTQ_PC: 1e-2, MODE_INT8_CB: 1e-2,
       MODE_SPEC: 2e-3, MODE_CHUNKED_PREFILL: 2e-3, MODE_CUDA_GRAPHS: 2e-3}
ORACLE_MODE = {MODE_FP16: 0, MODE_INT8: 1, MODE_GPTQ4: 2, MODE_AWQ4: 3, MODE_KV_COMPRESSION: 9, MODE_GPTQ_PC: 2, MODE_INT8_CB: 1,
               MODE_CHUNKED_PREFILL: 0, MODE_CUDA_GRAPHS: 0}


def prompt(seed, n, vocab):
    return (np.random.default_rng(seed).integers(0, vocab, size=n)).astype(np.int32)


@pytest.fixture(scope="module", params=["tiny", "tiny128"])
def pair(request, cuda_ok):
    shape = request.param
    cfg = engine_cfg(target=shape, draft="tiny_draft", seed=5, kv_blocks=512, max_seq_len=1024)
    eng = Engine(cfg)
    orc = O.OracleModel(model_cfg(shape), seed=5, max_ctx=1024)
    drf = O.OracleModel(model_cfg("tiny_draft"), seed=5, is_draft=True, max_ctx=1024)
    yield shape, eng, orc, drf
    eng.close()


def _check_logits(gpu, ref, tol):
    err = np.abs(gpu - ref).max(axis=1) / ref.std(axis=1)
    assert err.max() < tol, f"logit error {err.max():.3g} >= {tol}"


@pytest.mark.parametrize("mode", [MODE_FP16, MODE_INT8, MODE_GPTQ4, MODE_AWQ4, MODE_CHUNKED_PREFILL,
                                  MODE_CUDA_GRAPHS, MODE_KV_COMPRESSION])
@pytest.mark.parametrize("plen,n_new", [(1, 4), (37, 24), (130, 9)])
def test_batch1_modes_match_oracle(pair, mode, plen, n_new):
    _, eng, orc, _ = pair
    p = prompt(plen * 31 + mode, plen, eng.vocab)
    r = eng.run(mode, p, n_new, want_logits=True)
    toks, lg = orc.generate(ORACLE_MODE[mode], p, n_new, want_logits=True)
    assert np.array_equal(r.tokens, toks)
    _check_logits(r.logits, lg, TOL[mode])


@pytest.mark.parametrize("mode", [MODE_FP16, MODE_INT8, MODE_GPTQ4, MODE_AWQ4, MODE_KV_COMPRESSION])
def test_graph_replay_equals_oracle_tokens(pair, mode):
    _, eng, orc, _ = pair
    p = prompt(99 + mode, 50, eng.vocab)
    r = eng.run(mode, p, 40)  # no logits requested -> CUDA-graph decode loop
    toks, _ = orc.generate(ORACLE_MODE[mode], p, 40)
    assert np.array_equal(r.tokens, toks)
    assert r.kernel_launches > 0


def test_speculative_matches_target_greedy(pair):
    _, eng, orc, drf = pair
    p = prompt(7, 45, eng.vocab)
    r = eng.run(MODE_SPEC, p, 60, want_logits=True)
    toks, lg, st = O.spec_generate(orc, drf, 4, p, 60, want_logits=True)
    assert np.array_equal(r.tokens, toks)
    assert (r.spec_rounds, r.spec_proposed, r.spec_accepted) == (st["rounds"], st["proposed"], st["accepted"])
    assert 0 < r.spec_accepted < r.spec_proposed
    _check_logits(r.logits, lg, TOL[MODE_SPEC])
    greedy, _ = orc.generate(0, p, 60)
    assert np.array_equal(r.tokens, greedy)


@pytest.mark.parametrize("plen,n_new", [(1, 1), (1, 2), (3, 9), (45, 60), (200, 33)])
def test_speculative_device_loop(pair, plen, n_new):
    """The graph path (no logits requested: one WHILE-node graph launch per
    request, accept on the device) emits the target's greedy tokens with the
    oracle's round / accept counts, including n_new = 1 (no round) and 2."""
    _, eng, orc, drf = pair
    p = prompt(plen * 13 + n_new, plen, eng.vocab)
    r = eng.run(MODE_SPEC, p, n_new)
    toks, _, st = O.spec_generate(orc, drf, 4, p, n_new)
    assert np.array_equal(r.tokens, toks)
    assert (r.spec_rounds, r.spec_proposed, r.spec_accepted) == (st["rounds"], st["proposed"], st["accepted"])
    r2 = eng.run(MODE_SPEC, p, n_new)  # replay is stateless across requests
    assert np.array_equal(r2.tokens, toks) and r2.spec_rounds == r.spec_rounds


def test_speculative_eager_engine(cuda_ok):
    """use_graphs = 0: the same device round runs eagerly with a host check per round."""
    shape = "tiny"
    eng = Engine(engine_cfg(target=shape, draft="tiny_draft", seed=5, kv_blocks=256,
                            max_seq_len=512, use_graphs=0))
    orc = O.OracleModel(model_cfg(shape), seed=5, max_ctx=512)
    drf = O.OracleModel(model_cfg("tiny_draft"), seed=5, is_draft=True, max_ctx=512)
    p = prompt(71, 30, eng.vocab)
    r = eng.run(MODE_SPEC, p, 41)
    toks, _, st = O.spec_generate(orc, drf, 4, p, 41)
    eng.close()
    assert np.array_equal(r.tokens, toks)
    assert (r.spec_rounds, r.spec_accepted) == (st["rounds"], st["accepted"])


def test_prefix_caching_reuses_blocks_and_keeps_tokens(pair):
    _, eng, orc, _ = pair
    eng.reset_prefix_cache()
    shared = prompt(1234, 96, eng.vocab)
    outs = []
    for i in range(3):
        tail = prompt(2000 + i, 20 + i, eng.vocab)
        p = np.concatenate([shared, tail])
        r = eng.run(MODE_GPTQ_PC, p, 12, want_logits=True)
        toks, lg = orc.generate(2, p, 12, want_logits=True)
        assert np.array_equal(r.tokens, toks)
        _check_logits(r.logits, lg, TOL[MODE_GPTQ_PC])
        outs.append(r.prefix_hit_tokens)
    assert outs[0] == 0
    assert outs[1] == 96 and outs[2] == 96  # 6 full shared blocks reused


def test_continuous_batching_ragged_cohort(pair):
    _, eng, orc, _ = pair
    rng = np.random.default_rng(3)
    plens = [int(x) for x in rng.integers(5, 90, size=11)]
    nnew = [int(x) for x in rng.integers(1, 30, size=11)]
    prompts = [prompt(500 + i, plens[i], eng.vocab) for i in range(11)]
    res = eng.run_batch(MODE_INT8_CB, prompts, nnew, want_logits=True)
    for i, r in enumerate(res):
        toks, lg = orc.generate(1, prompts[i], nnew[i], want_logits=True)
        assert np.array_equal(r.tokens, toks), i
        _check_logits(r.logits, lg, TOL[MODE_INT8_CB])


def test_error_codes(pair):
    _, eng, _, _ = pair
    with pytest.raises(MswError) as e:
        eng.run(MODE_FP16, np.array([eng.vocab + 5], dtype=np.int32), 2)
    assert e.value.code == 3
    with pytest.raises(MswError) as e:
        eng.run(12, np.array([1, 2, 3], dtype=np.int32), 2)  # not an InferenceMode id
    assert e.value.code == 2
    with pytest.raises(MswError) as e:
        eng.run(MODE_FP16, np.arange(10, dtype=np.int32), 5000)
    assert e.value.code == 3


@pytest.fixture(scope="module")
def long_pair(cuda_ok):
    cfg = engine_cfg(target="tiny128", draft=None, seed=11, kv_blocks=2048, max_seq_len=4096)
    eng = Engine(cfg)
    orc = O.OracleModel(model_cfg("tiny128"), seed=11, max_ctx=4096)
    yield eng, orc
    eng.close()


@pytest.mark.parametrize("mode", [MODE_FP16, MODE_INT8])
def test_long_prefill_crosses_chunks(long_pair, mode):
    # 2100-token prompt: tensor-core prefill attention over 33 KV tiles, and a
    # second 2048-token prefill chunk reading the first chunk's paged K/V
    eng, orc = long_pair
    p = prompt(77 + mode, 2100, eng.vocab)
    r = eng.run(mode, p, 6, want_logits=True)
    toks, lg = orc.generate(ORACLE_MODE[mode], p, 6, want_logits=True)
    assert np.array_equal(r.tokens, toks)
    _check_logits(r.logits, lg, TOL[mode])


def test_continuous_batching_packed_prefill_straddles_chunks(long_pair):
    # ~2.8K prompt tokens packed into two prefill chunks; sequences straddle the
    # chunk boundary and tensor-core attention windows hold several sequences
    eng, orc = long_pair
    rng = np.random.default_rng(21)
    plens = [int(x) for x in rng.integers(150, 420, size=10)]
    nnew = [int(x) for x in rng.integers(2, 12, size=10)]
    prompts = [prompt(900 + i, plens[i], eng.vocab) for i in range(10)]
    res = eng.run_batch(MODE_INT8_CB, prompts, nnew, want_logits=True)
    for i, r in enumerate(res):
        toks, lg = orc.generate(1, prompts[i], nnew[i], want_logits=True)
        assert np.array_equal(r.tokens, toks), i
        _check_logits(r.logits, lg, TOL[MODE_INT8_CB])


def test_continuous_batching_more_requests_than_rows(long_pair):
    # 70 requests > 64 block-table rows: admission waits for retirements
    eng, orc = long_pair
    rng = np.random.default_rng(5)
    plens = [int(x) for x in rng.integers(3, 24, size=70)]
    nnew = [int(x) for x in rng.integers(1, 6, size=70)]
    prompts = [prompt(3000 + i, plens[i], eng.vocab) for i in range(70)]
    res = eng.run_batch(MODE_INT8_CB, prompts, nnew)
    for i, r in enumerate(res):
        toks, _ = orc.generate(1, prompts[i], nnew[i])
        assert np.array_equal(r.tokens, toks), i


def test_chunked_prefill_mode_512_token_chunks(long_pair):
    # ChunkedPrefill screening mode: a 1300-token prompt prefilled as 512+512+276,
    # each chunk attending to the earlier chunks' paged K/V
    eng, orc = long_pair
    p = prompt(4242, 1300, eng.vocab)
    r = eng.run(MODE_CHUNKED_PREFILL, p, 8, want_logits=True)
    toks, lg = orc.generate(0, p, 8, want_logits=True)
    assert np.array_equal(r.tokens, toks)
    _check_logits(r.logits, lg, TOL[MODE_CHUNKED_PREFILL])
    assert np.array_equal(eng.run(MODE_FP16, p, 8).tokens, toks)


def test_cuda_graphs_mode_on_eager_engine(cuda_ok):
    # engine configured eager: FP16 decodes with per-kernel launches, the
    # CudaGraphs screening mode replays the captured decode graph; same tokens
    cfg = engine_cfg(target="tiny", draft=None, modes=(MODE_FP16, MODE_CUDA_GRAPHS), seed=5,
                     kv_blocks=256, max_seq_len=512, use_graphs=False)
    eng = Engine(cfg)
    try:
        orc = O.OracleModel(model_cfg("tiny"), seed=5, max_ctx=512)
        p = prompt(31337, 40, eng.vocab)
        toks, _ = orc.generate(0, p, 30)
        rg = eng.run(MODE_CUDA_GRAPHS, p, 30)
        re_ = eng.run(MODE_FP16, p, 30)
        assert np.array_equal(rg.tokens, toks)
        assert np.array_equal(re_.tokens, toks)
        assert not eng.has_mode(MODE_INT8)
    finally:
        eng.close()


def test_continuous_batching_bitwise_deterministic(long_pair):
    # 40 live rows run the tcgen05 kind::i8 GEMM with split-K every step; the
    # split partials are combined in a fixed order (int32), so logits repeat
    # bit for bit across runs
    eng, _ = long_pair
    rng = np.random.default_rng(8)
    plens = [int(x) for x in rng.integers(20, 200, size=40)]
    nnew = [int(x) for x in rng.integers(3, 16, size=40)]
    prompts = [prompt(7000 + i, plens[i], eng.vocab) for i in range(40)]
    runs = [eng.run_batch(MODE_INT8_CB, prompts, nnew, want_logits=True) for _ in range(3)]
    for rr in runs[1:]:
        for a, b in zip(runs[0], rr):
            assert np.array_equal(a.tokens, b.tokens)
            assert np.array_equal(a.logits.view(np.uint32), b.logits.view(np.uint32))


def test_continuous_batching_waits_for_kv_blocks(cuda_ok):
    # a 12-block pool holds 2 of these 5-6-block sequences at a time:
    # admission waits for retirements instead of failing the cohort
    cfg = engine_cfg(target="tiny", draft=None, modes=(MODE_INT8, MODE_INT8_CB), seed=9,
                     kv_blocks=12, max_seq_len=256)
    eng = Engine(cfg)
    try:
        orc = O.OracleModel(model_cfg("tiny"), seed=9, max_ctx=256)
        prompts = [prompt(100 + i, 60 + i, eng.vocab) for i in range(12)]
        nnew = [12] * 12
        res = eng.run_batch(MODE_INT8_CB, prompts, nnew)
        for i, r in enumerate(res):
            toks, _ = orc.generate(1, prompts[i], nnew[i])
            assert np.array_equal(r.tokens, toks), i
        with pytest.raises(MswError) as e:  # one request larger than the whole pool
            eng.run_batch(MODE_INT8_CB, [prompt(1, 200, eng.vocab)], [50])
        assert e.value.code == 3
    finally:
        eng.close()


def test_kv_compression_runs_on_e4m3_cache(pair):
    """KV-cache compression (screening mode 9): the decode attends over an E4M3
    cache. Its logits match the oracle's E4M3-cache run far more closely than
    the FP16 run of the same request (so the compressed path really ran), the
    request's KV footprint is one byte per element, and repeated requests
    leave both block pools balanced (fp16 prefill blocks released after the
    conversion, E4M3 blocks at the end)."""
    _, eng, orc, _ = pair
    p = prompt(4242, 90, eng.vocab)
    ref, lg = orc.generate(9, p, 20, want_logits=True)
    _, lg16 = orc.generate(0, p, 20, want_logits=True)
    for _ in range(3):
        r = eng.run(MODE_KV_COMPRESSION, p, 20, want_logits=True)
        assert np.array_equal(r.tokens, ref)
    err = np.abs(r.logits - lg).max(axis=1) / lg.std(axis=1)
    e16 = np.abs(r.logits - lg16).max(axis=1) / lg16.std(axis=1)
    assert err.max() < TOL[MODE_KV_COMPRESSION]
    assert e16[1:].min() > 3 * err[1:].max(), f"KV-compressed run within reach of FP16: {e16} vs {err}"
    tokens = 110
    m16, m8 = eng.memory_bytes(MODE_FP16, tokens), eng.memory_bytes(MODE_KV_COMPRESSION, tokens)
    assert 2 * (m16 - m8) == m16 - eng.memory_bytes(MODE_FP16, 0)
