"""Back-to-back timeline of the two-CTA W4 decode GEMV (diagnostics build with
-DMSW_TRACE of gemv_w4.cu, e.g. scripts/build_variant.sh w4ctr ... ; run with
MSW_ENGINE_SO=libmsw_engine_w4ctr.so). Launches the chosen linears in a
repeating chain through msw_linear_decode (PDL), records per (launch, CTA)
globaltimer stamps, and prints per launch: first CTA start, consumers past
the PDL wait, first stage consumed, consumers done, last epilogue done
(medians / extremes over CTAs, us relative to the first launch's start), and
how many CTAs shared an SM with the previous launch."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_23057_b200._capi import check_engine, engine_lib  # noqa: E402

lib = engine_lib()
SHAPES = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096), "down": (4096, 14336)}
chain = [a for a in sys.argv[1:] if not a.startswith("--")] or ["qkv", "o", "gate_up", "down"]
bufs = {}
for name in set(chain):
    n, k = SHAPES[name]
    wb = n * k // 2
    bufs[name] = [(torch.randint(-2**31, 2**31 - 1, (wb // 4,), dtype=torch.int32, device="cuda"),
                   (torch.rand(n * (k // 128), device="cuda") * 1e-3).half()) for _ in range(3)]
x = torch.randn(14336, device="cuda") * 0.1
y = torch.empty(28672, device="cuda")
sp = torch.cuda.current_stream().cuda_stream
seq = (chain * 8)[:16]


def run():
    for i, name in enumerate(seq):
        n, k = SHAPES[name]
        w, s = bufs[name][i % 3]
        check_engine(lib.msw_linear_decode(2, w.data_ptr(), s.data_ptr(), n, k, x.data_ptr(), 1,
                                           y.data_ptr(), sp))


run()
torch.cuda.synchronize()
tr = torch.zeros(512 * 148 * 8, dtype=torch.int64, device="cuda")
assert lib.msw_w4c_trace_set(C.c_void_p(tr.data_ptr())) == 0
run()
torch.cuda.synchronize()
lib.msw_w4c_trace_set(C.c_void_p(0))
t = tr.cpu().numpy().reshape(512, 148, 8)
t0 = t[0, :, 1][t[0, :, 1] > 0].min()
prev_sm = None
print(f"chain {seq}")
for L in range(len(seq)):
    row = t[L]
    live = row[:, 1] > 0
    r = row[live]
    us = lambda c: (r[:, c] - t0) / 1000.0
    sm = r[:, 0]
    uniq, cnt = np.unique(sm, return_counts=True)
    doubled = np.isin(sm, uniq[cnt > 1])
    dbl = f"  sms {len(uniq)} doubled {int((cnt > 1).sum())}"
    if doubled.any() and (~doubled).any():
        dbl += f" cons_done(doubled) {np.median(us(4)[doubled]):7.2f} vs single {np.median(us(4)[~doubled]):7.2f}"
    print(f"{L:2d} {seq[L]:8s} start {us(1).min():7.2f}..{us(1).max():7.2f}  pdl_ok {np.median(us(2)):7.2f}  "
          f"first_stage {np.median(us(3)):7.2f}  cons_done {np.median(us(4)):7.2f} (max {us(4).max():7.2f})  "
          f"epi_done max {us(5).max():7.2f}  ctas {live.sum()}" + dbl)
