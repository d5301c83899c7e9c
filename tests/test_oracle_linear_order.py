"""The oracle's FP16 / W4 / AWQ4 linears are pinned bit-exactly to a numpy
restatement of their arithmetic contract (oracle_model.c, `dot8`): weights
dequantised to fp16 values (W4: fp16((q - z) * s_g)), x rounded to fp16,
products rounded to fp32 and added into eight lane accumulators (lane j
takes k = j mod 8, increasing k, no FMA), lanes summed in order from 0.
This pins the vectorised (AVX2 / F16C) oracle paths to the scalar contract
the GPU parity tolerances were set against. CPU only."""
import numpy as np
import pytest

import oracle as O


def dot8_rows(wf: np.ndarray, x16: np.ndarray) -> np.ndarray:
    n, k = wf.shape
    acc = np.zeros((n, 8), dtype=np.float32)
    for c in range(0, k, 8):
        acc = acc + (wf[:, c:c + 8] * x16[c:c + 8]).astype(np.float32)
    s = np.zeros(n, dtype=np.float32)
    for j in range(8):
        s = s + acc[:, j]
    return s


def w4_dequant(q: np.ndarray, s16: np.ndarray, z=None) -> np.ndarray:
    n, k = q.shape
    sc = s16.view(np.float16).astype(np.float32)
    zz = np.full(sc.shape, 8, dtype=np.int32) if z is None else z.astype(np.int32)
    v = (q.astype(np.int32).reshape(n, k // 128, 128) - zz[:, :, None]).astype(np.float32)
    return (v * sc[:, :, None]).astype(np.float16).astype(np.float32).reshape(n, k)


@pytest.mark.parametrize("n,k", [(48, 256), (130, 1024), (17, 4096)])
def test_linear_fp16_w4_awq4_match_dot8_contract(n, k):
    rng = np.random.default_rng(n * 7 + k)
    x = (rng.standard_normal((2, k)) * 1.5).astype(np.float32)
    x16 = x.astype(np.float16).astype(np.float32)
    w16 = (rng.standard_normal((n, k)) * 0.05).astype(np.float16)
    w16[0, :8] = np.arange(1, 9, dtype=np.uint16).view(np.float16)  # fp16 denormals
    y = O.linear(0, w16.view(np.uint16), None, x)
    ref = np.stack([dot8_rows(w16.astype(np.float32), x16[t]) for t in range(2)])
    assert np.array_equal(y.view(np.uint32), ref.view(np.uint32))

    q = rng.integers(0, 16, (n, k), dtype=np.uint8)
    s16 = (10.0 ** rng.uniform(-6, -1, (n, k // 128)) * rng.choice([-1, 1], (n, k // 128)))
    s16 = s16.astype(np.float16).view(np.uint16)
    y = O.linear(2, q, s16, x)
    ref = np.stack([dot8_rows(w4_dequant(q, s16), x16[t]) for t in range(2)])
    assert np.array_equal(y.view(np.uint32), ref.view(np.uint32))

    z = rng.integers(0, 16, (n, k // 128), dtype=np.uint8)
    y = O.linear_awq4(q, s16, z, x)
    ref = np.stack([dot8_rows(w4_dequant(q, s16, z), x16[t]) for t in range(2)])
    assert np.array_equal(y.view(np.uint32), ref.view(np.uint32))
