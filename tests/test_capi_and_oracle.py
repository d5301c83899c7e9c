"""CPU checks of the boundary and the checker:
  * both C-ABI libraries load (no GPU needed) and export every function that
    include/msw_engine.h and include/msw_host.h declare;
  * the CPU oracle's internal invariants (speculative decoding == target
    greedy, successor init, quantiser round trips, INT8 exactness bounds).
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle as O
from paper_2605_23057_b200 import _capi
from paper_2605_23057_b200.configs import model_cfg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(msw_[a-z0-9_]+)\s*\(", text)))


@pytest.mark.parametrize("header,loader", [("msw_engine.h", _capi.engine_lib),
                                           ("msw_host.h", _capi.host_lib)])
def test_library_exports_every_declared_symbol(header, loader):
    lib = loader()
    names = _declared(header)
    assert len(names) >= 7
    for n in names:
        assert hasattr(lib, n), f"{n} declared in {header} but not exported"


def test_engine_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2605_23057_b200.engine import Engine
    with pytest.raises(_capi.MswError) as e:
        Engine(target="tiny", draft="tiny_draft")
    assert e.value.code == 1


@pytest.fixture(scope="module")
def tiny():
    m = O.OracleModel(model_cfg("tiny"), seed=3, max_ctx=512)
    d = O.OracleModel(model_cfg("tiny_draft"), seed=3, is_draft=True, agree_permille=700,
                      max_ctx=512)
    return m, d


def test_oracle_successor_init_is_peaked(tiny):
    m, _ = tiny
    p = np.arange(10, dtype=np.int32) * 7
    for mode in (0, 1, 2):
        toks, lg = m.generate(mode, p, 12, want_logits=True)
        s = np.sort(lg, axis=1)
        assert ((s[:, -1] - s[:, -2]) / lg.std(axis=1)).min() > 5.0  # argmax robust to fp error
        assert all(toks[i + 1] == m.successor(toks[i]) for i in range(11))


def test_oracle_spec_equals_target_greedy(tiny):
    m, d = tiny
    p = (np.arange(33, dtype=np.int32) * 13 + 1) % 2048
    toks, _, st = O.spec_generate(m, d, 4, p, 50)
    greedy, _ = m.generate(0, p, 50)
    assert np.array_equal(toks, greedy)
    assert st["proposed"] == 4 * st["rounds"] and 0 < st["accepted"] < st["proposed"]


def test_oracle_quantisers():
    w = O.fill_fp16(16, 256, 1, 42, 4)
    q8, s8 = O.quant_int8_rows(w)
    wf = w.view(np.float16).astype(np.float32)
    assert np.abs(q8).max() <= 127
    assert np.abs(q8 * s8[:, None] - wf).max() <= s8.max() * 0.5 + 1e-7
    q4, s4 = O.quant_w4_rows(w)
    assert q4.min() >= 0 and q4.max() <= 15
    deq = (q4.astype(np.float32) - 8).reshape(16, 2, 128) * s4.view(np.float16).astype(np.float32)[:, :, None]
    assert np.abs(deq.reshape(16, 256) - wf).max() <= s4.view(np.float16).astype(np.float32).max() * 0.51


def test_int8_accumulators_cannot_overflow():
    # |acc| <= 127^2 * K for the largest K in the 8B shape (FFN 14336) < 2^31
    assert 127 * 127 * 14336 < 2 ** 31
    w = np.full((2, 14336), 127, dtype=np.int8)
    x = np.full(14336, 127, dtype=np.int8)
    assert O.gemv_i8_acc(w, x)[0] == 127 * 127 * 14336
