"""CPU ORACLE wrapper — TEST INFRASTRUCTURE ONLY.

ctypes binding of oracle/liboracle.so (the C restatement in oracle_model.c).
Imported only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
and --impl reference legs, as the checker. The product (paper_2605_23057_b200)
never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make -C oracle`")
        L = C.CDLL(path)
        vp, i32, i64, u64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64
        L.orc_model_create.restype = vp
        L.orc_model_create.argtypes = [vp, u64, C.c_int, i32, C.c_uint32, i32]
        L.orc_model_destroy.argtypes = [vp]
        L.orc_generate.argtypes = [vp, C.c_int, vp, C.c_int, C.c_int, vp, vp]
        L.orc_spec_generate.argtypes = [vp, vp, C.c_int, vp, C.c_int, C.c_int, vp, vp, vp, vp, vp]
        L.orc_successor.argtypes = [vp, i32]
        L.orc_successor.restype = i32
        L.orc_fill_fp16.argtypes = [vp, i64, i64, u64, u64, i32]
        L.orc_quant_int8_rows.argtypes = [vp, i32, i32, vp, vp]
        L.orc_quant_w4_rows.argtypes = [vp, i32, i32, vp, vp]
        L.orc_gemv_i8_acc.argtypes = [vp, vp, i32, i32, vp]
        L.orc_linear.argtypes = [C.c_int, vp, vp, i32, i32, vp, i32, vp]
        L.orc_model_tensor.argtypes = [vp, C.c_int, C.c_int, C.c_int, vp, vp]
        L.orc_quant_awq4_rows.argtypes = [vp, i32, i32, vp, vp, vp]
        L.orc_linear_awq4.argtypes = [vp, vp, vp, i32, i32, vp, i32, vp]
        L.orc_fp8_e4m3_roundtrip.argtypes = [vp, C.c_int64, vp, vp]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class OracleModel:
    def __init__(self, cfg, seed: int = 0, is_draft: bool = False, agree_permille: int = 800,
                 modes_mask: int = 0xFFF, max_ctx: int = 2048):
        self.cfg = cfg
        self.vocab = cfg.vocab
        self.h = lib().orc_model_create(C.byref(cfg), seed, int(is_draft), agree_permille,
                                        modes_mask, max_ctx)
        if not self.h:
            raise RuntimeError("orc_model_create failed")

    def close(self):
        if self.h:
            lib().orc_model_destroy(self.h)
            self.h = None

    __del__ = close

    def generate(self, mode: int, prompt, n_new: int, want_logits: bool = False):
        p = np.ascontiguousarray(prompt, dtype=np.int32)
        out = np.zeros(n_new, dtype=np.int32)
        lg = np.zeros((n_new, self.vocab), dtype=np.float32) if want_logits else None
        rc = lib().orc_generate(self.h, mode, _p(p), len(p), n_new, _p(out),
                                _p(lg) if lg is not None else None)
        if rc != 0:
            raise RuntimeError(f"orc_generate failed rc={rc}")
        return out, lg

    def successor(self, t: int) -> int:
        return lib().orc_successor(self.h, int(t))

    # tensor ids of orc_model_tensor (oracle_model.h)
    EMBED, LM_HEAD, FINAL_NORM, ATTN_NORM, FFN_NORM, QKV, O, GATE, UP, DOWN = range(10)

    def tensor(self, which: int, layer: int = 0, fmt: int = 0):
        """One weight tensor: fp16 array (fmt 0 / norms / embed / lm_head), or
        (q int8 [n,k], s fp32 [n]) for fmt 1, (q nibble-per-byte [n,k], s fp16
        [n,k/128]) for fmt 2 (GPTQ4) and 3 (AWQ4); fmt 4: AWQ4 zeros [n,k/128]."""
        c = self.cfg
        H, V, F, D = c.hidden, c.vocab, c.ffn, c.head_dim
        if which in (self.EMBED, self.LM_HEAD):
            shape = (V, H)
        elif which in (self.FINAL_NORM, self.ATTN_NORM, self.FFN_NORM):
            shape = (H,)
        else:
            shape = {self.QKV: ((c.n_heads + 2 * c.n_kv_heads) * D, H), self.O: (H, c.n_heads * D),
                     self.GATE: (F, H), self.UP: (F, H), self.DOWN: (H, F)}[which]
        if which < self.QKV or fmt == 0:
            w = np.zeros(shape, np.float16)
            s = None
        elif fmt == 1:
            w, s = np.zeros(shape, np.int8), np.zeros(shape[0], np.float32)
        elif fmt == 4:  # AWQ4 zero points
            w, s = np.zeros((shape[0], shape[1] // 128), np.uint8), None
        else:
            w, s = np.zeros(shape, np.uint8), np.zeros((shape[0], shape[1] // 128), np.float16)
        rc = lib().orc_model_tensor(self.h, which, layer, fmt, _p(w), _p(s) if s is not None else None)
        if rc != 0:
            raise RuntimeError(f"orc_model_tensor({which}, {layer}, {fmt}) not resident")
        return w if s is None else (w, s)


def spec_generate(target: OracleModel, draft: OracleModel, k: int, prompt, n_new: int,
                  want_logits: bool = False):
    p = np.ascontiguousarray(prompt, dtype=np.int32)
    out = np.zeros(n_new, dtype=np.int32)
    lg = np.zeros((n_new, target.vocab), dtype=np.float32) if want_logits else None
    r, pr, ac = C.c_int32(), C.c_int32(), C.c_int32()
    rc = lib().orc_spec_generate(target.h, draft.h, k, _p(p), len(p), n_new, _p(out),
                                 _p(lg) if lg is not None else None,
                                 C.byref(r), C.byref(pr), C.byref(ac))
    if rc != 0:
        raise RuntimeError(f"orc_spec_generate failed rc={rc}")
    return out, lg, dict(rounds=r.value, proposed=pr.value, accepted=ac.value)


def fill_fp16(rows: int, cols: int, seed: int, tensor_id: int, scale_log2: int) -> np.ndarray:
    a = np.zeros((rows, cols), dtype=np.uint16)
    lib().orc_fill_fp16(_p(a), rows, cols, seed, tensor_id, scale_log2)
    return a


def quant_int8_rows(w: np.ndarray):
    n, k = w.shape
    q = np.zeros((n, k), dtype=np.int8)
    s = np.zeros(n, dtype=np.float32)
    lib().orc_quant_int8_rows(_p(np.ascontiguousarray(w)), n, k, _p(q), _p(s))
    return q, s


def quant_w4_rows(w: np.ndarray):
    n, k = w.shape
    q = np.zeros((n, k), dtype=np.uint8)
    s = np.zeros((n, k // 128), dtype=np.uint16)
    lib().orc_quant_w4_rows(_p(np.ascontiguousarray(w)), n, k, _p(q), _p(s))
    return q, s


def quant_awq4_rows(w: np.ndarray):
    """AWQ format: q nibble-per-byte [n,k], fp16-bit scales and uint8 zeros [n,k/128]."""
    n, k = w.shape
    q = np.zeros((n, k), dtype=np.uint8)
    s = np.zeros((n, k // 128), dtype=np.uint16)
    z = np.zeros((n, k // 128), dtype=np.uint8)
    lib().orc_quant_awq4_rows(_p(np.ascontiguousarray(w)), n, k, _p(q), _p(s), _p(z))
    return q, s, z


def linear_awq4(q: np.ndarray, s: np.ndarray, z: np.ndarray, x: np.ndarray) -> np.ndarray:
    n, k = q.shape
    x = np.ascontiguousarray(x, dtype=np.float32).reshape(-1, k)
    y = np.zeros((x.shape[0], n), dtype=np.float32)
    lib().orc_linear_awq4(_p(np.ascontiguousarray(q)), _p(np.ascontiguousarray(s)),
                          _p(np.ascontiguousarray(z)), n, k, _p(x), x.shape[0], _p(y))
    return y


def fp8_e4m3(x16: np.ndarray):
    """fp16 bits (uint16) -> (E4M3 bytes, their fp16 bits): RNE, saturating."""
    x16 = np.ascontiguousarray(x16, dtype=np.uint16).ravel()
    q = np.zeros(x16.size, dtype=np.uint8)
    y = np.zeros(x16.size, dtype=np.uint16)
    lib().orc_fp8_e4m3_roundtrip(_p(x16), x16.size, _p(q), _p(y))
    return q, y


def gemv_i8_acc(w: np.ndarray, x: np.ndarray) -> np.ndarray:
    n, k = w.shape
    acc = np.zeros(n, dtype=np.int32)
    lib().orc_gemv_i8_acc(_p(np.ascontiguousarray(w)), _p(np.ascontiguousarray(x)), n, k, _p(acc))
    return acc


def linear(wtype: int, w: np.ndarray, scales, x: np.ndarray) -> np.ndarray:
    """y[t, n]; w fp16 bits uint16 [n,k] / int8 [n,k] / W4 nibble-per-byte [n,k]."""
    n, k = w.shape
    x = np.ascontiguousarray(x, dtype=np.float32).reshape(-1, k)
    y = np.zeros((x.shape[0], n), dtype=np.float32)
    lib().orc_linear(wtype, _p(np.ascontiguousarray(w)),
                     _p(np.ascontiguousarray(scales)) if scales is not None else None,
                     n, k, _p(x), x.shape[0], _p(y))
    return y
