"""Kernel-level parity on the B200: every sm_100a kernel called through the C
ABI (device pointers from torch) against the CPU oracle on the same inputs.

Bars: K16 init, W8 and W4 quantisers and the INT8 int32 accumulator are
BIT-EXACT; FP16 / W4 / W8A8 linears (decode GEMV for t <= 6, tcgen05 GEMM
for t > 6 and n % 128 == 0, CUDA-core tile GEMM otherwise) within the stated
relative tolerance
(max |gpu - oracle| / max |oracle|):  FP16 2e-5 (GEMV) / 1e-4 (tcgen05
accumulation over K up to 14336), W4 2e-3 (fp16 partial sums of <= 4
products by contract). W8A8 linears are BIT-EXACT end to end
(same per-token quantisation, exact int32 accumulators, the same two scale
multiplies), and msw_linear_i8_raw exposes the production kernels' int32
accumulators for a direct comparison."""
import ctypes as C

import numpy as np
import pytest

import oracle as O
from paper_2605_23057_b200 import _capi
from paper_2605_23057_b200._capi import check_engine, engine_lib

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    return torch


def _pack_w4_host(q):
    """Reference packing of nibble-per-byte q [n,k] into the engine layout
    (word j = k 8j..8j+7, nibble position p(i) = (i>>1) + 4*(i&1))."""
    n, k = q.shape
    qq = q.reshape(n, k // 8, 8).astype(np.uint32)
    pos = np.array([(i >> 1) + 4 * (i & 1) for i in range(8)], dtype=np.uint32)
    return (qq << (4 * pos)).sum(axis=2).astype(np.uint32)


@pytest.mark.parametrize("rows,cols,tid,shift", [(64, 512, 17, 5), (3, 4096, 1 << 32, 6), (128, 384, 259, 0)])
def test_fill_fp16_bit_exact(cuda_ok, rows, cols, tid, shift):
    torch = _torch()
    d = torch.empty((rows, cols), dtype=torch.int16, device="cuda")
    check_engine(engine_lib().msw_fill_fp16(d.data_ptr(), rows, cols, 7, tid, shift, None))
    torch.cuda.synchronize()
    ref = O.fill_fp16(rows, cols, 7, tid, shift)
    assert np.array_equal(d.cpu().numpy().view(np.uint16), ref)


def test_quantisers_bit_exact(cuda_ok):
    torch = _torch()
    n, k = 96, 1024
    w = O.fill_fp16(n, k, 3, 99, 6)
    w[5, :] = 0  # all-zero row: scale 0, q = 0 / 8
    dw = torch.from_numpy(w.view(np.int16)).cuda()
    q8 = torch.empty((n, k), dtype=torch.int8, device="cuda")
    s8 = torch.empty(n, dtype=torch.float32, device="cuda")
    check_engine(engine_lib().msw_quant_int8_rows(dw.data_ptr(), n, k, q8.data_ptr(), s8.data_ptr(), None))
    q4 = torch.empty((n, k // 8), dtype=torch.int32, device="cuda")
    s4 = torch.empty((n, k // 128), dtype=torch.int16, device="cuda")
    check_engine(engine_lib().msw_quant_w4_rows(dw.data_ptr(), n, k, q4.data_ptr(), s4.data_ptr(), None))
    torch.cuda.synchronize()
    rq8, rs8 = O.quant_int8_rows(w)
    rq4, rs4 = O.quant_w4_rows(w)
    assert np.array_equal(q8.cpu().numpy(), rq8)
    assert np.array_equal(s8.cpu().numpy().view(np.uint32), rs8.view(np.uint32))
    assert np.array_equal(q4.cpu().numpy().view(np.uint32), _pack_w4_host(rq4))
    assert np.array_equal(s4.cpu().numpy().view(np.uint16), rs4)


@pytest.mark.parametrize("n,k", [(256, 4096), (130, 14336), (8, 16)])
def test_int8_accumulators_bit_exact(cuda_ok, n, k):
    torch = _torch()
    rng = np.random.default_rng(n + k)
    w = rng.integers(-127, 128, size=(n, k), dtype=np.int8)
    x = rng.integers(-127, 128, size=k, dtype=np.int8)
    w[0, :] = 127
    x[:] = np.where(np.arange(k) % 2 == 0, 127, x)  # near-extreme sums
    acc = torch.empty(n, dtype=torch.int32, device="cuda")
    dw, dx = torch.from_numpy(w).cuda(), torch.from_numpy(x).cuda()  # keep alive across the call
    check_engine(engine_lib().msw_gemv_i8_acc(dw.data_ptr(), dx.data_ptr(), n, k, acc.data_ptr(),
                                              None))
    torch.cuda.synchronize()
    assert np.array_equal(acc.cpu().numpy(), O.gemv_i8_acc(w, x))


def _run_linear(fmt, w_dev, s_dev, n, k, x):
    torch = _torch()
    t = x.shape[0]
    dx = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()
    dy = torch.empty((t, n), dtype=torch.float32, device="cuda")
    check_engine(engine_lib().msw_linear(fmt, w_dev.data_ptr(), s_dev.data_ptr() if s_dev is not None else None,
                                         n, k, dx.data_ptr(), t, dy.data_ptr(), None))
    torch.cuda.synchronize()
    return dy.cpu().numpy()


@pytest.mark.parametrize("t", [1, 2, 5, 6, 7, 40, 129, 300])
@pytest.mark.parametrize("n,k", [(512, 4096), (2048, 512), (256, 14336), (96, 256)])
def test_linear_formats_vs_oracle(cuda_ok, t, n, k):
    torch = _torch()
    rng = np.random.default_rng(t * 1000 + n)
    w = O.fill_fp16(n, k, 11, 1234 + n, (int(np.ceil(np.log2(k))) + 1) // 2)
    x = rng.standard_normal((t, k)).astype(np.float32)
    x[:, 0] = 4.0  # a large activation, as after RMSNorm with outliers
    # FP16
    y = _run_linear(_capi.W_FP16, torch.from_numpy(w.view(np.int16)).cuda(), None, n, k, x)
    ref = O.linear(_capi.W_FP16, w, None, x)
    tol_fp = 2e-5 if t <= 6 else 1e-4  # tensor-core (tcgen05) fp32 accumulation for t > 6
    assert np.abs(y - ref).max() / np.abs(ref).max() < tol_fp
    # W8A8
    q8, s8 = O.quant_int8_rows(w)
    y = _run_linear(_capi.W_INT8, torch.from_numpy(q8).cuda(), torch.from_numpy(s8).cuda(), n, k, x)
    ref = O.linear(_capi.W_INT8, q8, s8, x)
    assert np.array_equal(y, ref)  # exact int32 accumulators, identical scale multiplies
    # W4 g128
    q4, s4 = O.quant_w4_rows(w)
    packed = _pack_w4_host(q4)
    y = _run_linear(_capi.W_W4, torch.from_numpy(packed.view(np.int32)).cuda(),
                    torch.from_numpy(s4.view(np.int16)).cuda(), n, k, x)
    ref = O.linear(_capi.W_W4, q4, s4, x)
    assert np.abs(y - ref).max() / np.abs(ref).max() < 2e-3


def _i8_raw(w, x):
    torch = _torch()
    n, k = w.shape
    t = x.shape[0]
    dw = torch.from_numpy(np.ascontiguousarray(w)).cuda()
    dx = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()
    acc = torch.empty((t, n), dtype=torch.int32, device="cuda")
    check_engine(engine_lib().msw_linear_i8_raw(dw.data_ptr(), n, k, dx.data_ptr(), t, acc.data_ptr(), None))
    torch.cuda.synchronize()
    return acc.cpu().numpy()


@pytest.mark.parametrize("t", [1, 2, 5, 6, 7, 64, 300])
@pytest.mark.parametrize("n,k", [(4096, 4096), (1024, 14336), (256, 4096), (96, 512)])
def test_int8_production_accumulators_bit_exact(cuda_ok, t, n, k):
    """The W8A8 product kernels (decode GEMV t<=6, tcgen05 kind::i8 GEMM with
    its deterministic split-K t>6, tile GEMM for n % 128 != 0) return int32
    accumulators identical to the oracle's exact integer dot products."""
    rng = np.random.default_rng(t * 7919 + n + k)
    w = rng.integers(-127, 128, size=(n, k), dtype=np.int8)
    w[0, :] = 127  # row at the int32 extreme: 127*127*k
    xi = rng.integers(-127, 128, size=(t, k)).astype(np.int8)
    xi[:, 0] = 127  # absmax 127 -> per-token scale 1, quantisation is the identity
    xi[0, :] = 127
    got = _i8_raw(w, xi.astype(np.float32))
    ref = np.stack([O.gemv_i8_acc(w, xi[i]) for i in range(t)])
    assert np.array_equal(got, ref)


def test_int8_split_k_linear_deterministic(cuda_ok):
    """The tcgen05 INT8 linear at a continuous-batching shape (T=64, split-K 4)
    is bitwise identical across repeated launches and equals the oracle."""
    torch = _torch()
    n, k, t = 4096, 4096, 64
    w = O.fill_fp16(n, k, 5, 4242, 6)
    q8, s8 = O.quant_int8_rows(w)
    x = np.random.default_rng(1).standard_normal((t, k)).astype(np.float32)
    dq, ds = torch.from_numpy(q8).cuda(), torch.from_numpy(s8).cuda()
    outs = [_run_linear(_capi.W_INT8, dq, ds, n, k, x) for _ in range(8)]
    for o in outs[1:]:
        assert np.array_equal(o.view(np.uint32), outs[0].view(np.uint32))
    assert np.array_equal(outs[0], O.linear(_capi.W_INT8, q8, s8, x))


@pytest.mark.parametrize("n,k", [(4096, 4096), (6144, 4096), (4096, 14336), (2400, 4096)])
def test_w4_decode_balanced_ranges(cuda_ok, n, k):
    """Batch-1 W4 decode GEMV at 8B shapes (o, qkv, down, and an n where tiles
    do not divide evenly): with >= 148 tiles each CTA streams a chunk-balanced
    range and tiles straddling two CTAs are finished by the second one to
    arrive. Within the W4 bar of the oracle and bitwise identical across
    repeated launches (the two-part fp32 sum is order-independent)."""
    torch = _torch()
    w = O.fill_fp16(n, k, 3, 777 + n + k, (int(np.ceil(np.log2(k))) + 1) // 2)
    q4, s4 = O.quant_w4_rows(w)
    packed = _pack_w4_host(q4)
    dw = torch.from_numpy(packed.view(np.int32)).cuda()
    ds = torch.from_numpy(s4.view(np.int16)).cuda()
    x = np.random.default_rng(n + k).standard_normal((1, k)).astype(np.float32)
    outs = [_run_linear(_capi.W_W4, dw, ds, n, k, x) for _ in range(6)]
    for o in outs[1:]:
        assert np.array_equal(o.view(np.uint32), outs[0].view(np.uint32))
    ref = O.linear(_capi.W_W4, q4, s4, x)
    assert np.abs(outs[0] - ref).max() / np.abs(ref).max() < 2e-3


@pytest.mark.parametrize("fmt,t,n,k", [(_capi.W_FP16, 6, 256, 14336), (_capi.W_FP16, 5, 256, 14336),
                                       (_capi.W_FP16, 6, 512, 4096), (_capi.W_INT8, 6, 256, 14336),
                                       (_capi.W_INT8, 4, 512, 4096), (_capi.W_W4, 1, 4096, 14336)])
def test_decode_gemv_stress_repeatable(cuda_ok, fmt, t, n, k):
    """Repeated launches of the decode GEMV (one CTA per SM, cp.async.bulk ring
    read with generic loads) are bitwise identical and within the oracle bar.
    The FP16 6-token K=14336 shape leaves a 2-stage ring; it returned stale
    tiles in ~1.5% of runs until the producer fenced the consumers' generic
    reads against the async-proxy overwrite (fence.proxy.async, gemv.cu)."""
    torch = _torch()
    w = O.fill_fp16(n, k, 13, 999 + n + k, (int(np.ceil(np.log2(k))) + 1) // 2)
    lib = engine_lib()
    if fmt == _capi.W_FP16:
        src, s, ref_w, ref_s = torch.from_numpy(w.view(np.int16)).cuda(), None, w, None
    elif fmt == _capi.W_INT8:
        q8, s8 = O.quant_int8_rows(w)
        src, s, ref_w, ref_s = torch.from_numpy(q8).cuda(), torch.from_numpy(s8).cuda(), q8, s8
    else:
        q4, s4 = O.quant_w4_rows(w)
        src = torch.from_numpy(_pack_w4_host(q4).view(np.int32)).cuda()
        s, ref_w, ref_s = torch.from_numpy(s4.view(np.int16)).cuda(), q4, s4
    tf = torch.empty_like(src)
    check_engine(lib.msw_repack_decode(fmt, src.data_ptr(), n, k, tf.data_ptr(), None))
    x = np.random.default_rng(k + t).standard_normal((t, k)).astype(np.float32)
    dx = torch.from_numpy(x).cuda()
    outs = []
    for _ in range(60):
        dy = torch.full((t, n), float("nan"), device="cuda")
        check_engine(lib.msw_linear_decode(fmt, tf.data_ptr(), s.data_ptr() if s is not None else None,
                                           n, k, dx.data_ptr(), t, dy.data_ptr(), None))
        outs.append(dy)
    torch.cuda.synchronize()
    first = outs[0].cpu().numpy()
    for o in outs[1:]:
        assert np.array_equal(o.cpu().numpy().view(np.uint32), first.view(np.uint32))
    ref = O.linear(fmt, ref_w, ref_s, x)
    tol = {_capi.W_FP16: 2e-5, _capi.W_INT8: 0.0, _capi.W_W4: 2e-3}[fmt]
    assert np.abs(first - ref).max() <= tol * np.abs(ref).max()


def test_awq4_quantiser_bit_exact(cuda_ok):
    """msw_quant_awq4_rows (AWQ asymmetric g128: fp16 scale, uint8 zero point)
    packs the same nibbles, scales and zero points as the oracle's restatement
    of AutoAWQ pseudo_quantize (pinned in test_oracle_pin.py), including a
    constant group (max == min) and an all-zero row."""
    torch = _torch()
    n, k = 96, 1024
    w = O.fill_fp16(n, k, 3, 4321, 6)
    w[5, :] = 0
    w[7, 128:256] = w[7, 130]
    w[10:30] &= 0x7FFF  # all-positive rows: zero point 0
    w[30:50] |= 0x8000  # all-negative rows: zero point 15
    w[50:60, ::2] &= 0x7FFF  # skewed groups
    dw = torch.from_numpy(w.view(np.int16)).cuda()
    q = torch.empty((n, k // 8), dtype=torch.int32, device="cuda")
    s = torch.empty((n, k // 128), dtype=torch.int16, device="cuda")
    z = torch.empty((n, k // 128), dtype=torch.uint8, device="cuda")
    check_engine(engine_lib().msw_quant_awq4_rows(dw.data_ptr(), n, k, q.data_ptr(), s.data_ptr(),
                                                  z.data_ptr(), None))
    torch.cuda.synchronize()
    rq, rs, rz = O.quant_awq4_rows(w)
    assert np.array_equal(q.cpu().numpy().view(np.uint32), _pack_w4_host(rq))
    assert np.array_equal(s.cpu().numpy().view(np.uint16), rs)
    assert np.array_equal(z.cpu().numpy(), rz)
    assert rz.max() <= 15 and {0, 7, 8, 15} <= set(np.unique(rz).tolist())


@pytest.mark.parametrize("t", [1, 2, 5, 6, 7, 129, 300])
@pytest.mark.parametrize("n,k", [(512, 4096), (4096, 4096), (256, 14336), (96, 256), (2400, 4096)])
def test_linear_awq4_vs_oracle(cuda_ok, t, n, k):
    """AWQ4 linears (zero-point W4: decode GEMV t <= 6, tcgen05 GEMM with the
    packed-weight dequant producer t > 6 and n % 128 == 0, tile GEMM otherwise)
    against the oracle's (q - z) * s reference; the W4 bar (fp16 partial sums)."""
    torch = _torch()
    rng = np.random.default_rng(t * 17 + n + k)
    w = O.fill_fp16(n, k, 23, 5678 + n, (int(np.ceil(np.log2(k))) + 1) // 2)
    x = rng.standard_normal((t, k)).astype(np.float32)
    x[:, 0] = 4.0
    q, s, z = O.quant_awq4_rows(w)
    dq = torch.from_numpy(_pack_w4_host(q).view(np.int32)).cuda()
    ds = torch.from_numpy(s.view(np.int16)).cuda()
    dz = torch.from_numpy(z).cuda()
    dx = torch.from_numpy(x).cuda()
    dy = torch.empty((t, n), dtype=torch.float32, device="cuda")
    check_engine(engine_lib().msw_linear_awq4(dq.data_ptr(), ds.data_ptr(), dz.data_ptr(), n, k,
                                              dx.data_ptr(), t, dy.data_ptr(), None))
    torch.cuda.synchronize()
    y = dy.cpu().numpy()
    ref = O.linear_awq4(q, s, z, x)
    assert np.abs(y - ref).max() / np.abs(ref).max() < 2e-3


def test_fp8_e4m3_kv_rounding_bit_exact(cuda_ok):
    """The KV-cache compression mode's E4M3 rounding (cvt.rn.satfinite on the
    device) against the oracle's restatement (itself pinned to torch's
    float8_e4m3fn in test_oracle_pin.py) on every finite fp16 value: E4M3
    bytes and their fp16 widening bit-exact, |x| >= 464 saturating to 448."""
    torch = _torch()
    bits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    x = bits[np.isfinite(bits.view(np.float16))]
    x = x[: x.size // 2 * 2]
    dx = torch.from_numpy(x.view(np.int16)).cuda()
    q = torch.empty(x.size, dtype=torch.uint8, device="cuda")
    y = torch.empty(x.size, dtype=torch.int16, device="cuda")
    check_engine(engine_lib().msw_fp8_e4m3_roundtrip(dx.data_ptr(), x.size, q.data_ptr(), y.data_ptr(), None))
    torch.cuda.synchronize()
    rq, ry = O.fp8_e4m3(x)
    assert np.array_equal(q.cpu().numpy(), rq)
    assert np.array_equal(y.cpu().numpy().view(np.uint16), ry)
    big = np.abs(x.view(np.float16).astype(np.float32)) >= 464
    assert big.any() and np.all(np.abs(ry[big].view(np.float16).astype(np.float32)) == 448)
