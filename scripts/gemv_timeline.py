"""Intra-CTA timeline of the W4 decode GEMV from the diagnostics build
(libmsw_engine_trace.so, -DMSW_TRACE): per probe, the median / max over CTAs
of clock64 cycles since the producer's first probe, in us at 1.965 GHz.
Probes (gemv.cu): 0 producer start, 1 ring primed, 2 last stage issued,
3 consumers past griddepcontrol.wait, 4 activations staged, 5 first stage
consumed, 6 ring wrapped, 7 consumer warp 0 done, 8 first tile stored,
9 all tiles stored. Usage: gemv_timeline.py [shape] [--l2] [--back2back]."""
import ctypes as C
import os
import sys

os.environ.setdefault("MSW_ENGINE_SO", "libmsw_engine_trace.so")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_23057_b200._capi import check_engine, engine_lib  # noqa: E402

lib = engine_lib()
SHAPES = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096), "down": (4096, 14336)}
names = [a for a in sys.argv[1:] if not a.startswith("--")] or list(SHAPES)
NAMES = ["prod_start", "ring_primed", "last_issued", "cons_pdl_ok", "act_staged", "first_stage",
         "ring_wrap", "cons_done", "tile0_stored", "epi_done"]
for name in names:
    n, k = SHAPES[name]
    wb = n * k // 2
    copies = 1 if "--l2" in sys.argv else 4
    ws = [torch.randint(-2**31, 2**31 - 1, (wb // 4,), dtype=torch.int32, device="cuda") for _ in range(copies)]
    ss = [(torch.rand(n * (k // 128), device="cuda") * 1e-3).half() for _ in range(copies)]
    x = torch.randn(k, device="cuda") * 0.1
    y = torch.empty(n, device="cuda")
    buf = torch.zeros(148 * 16, dtype=torch.int64, device="cuda")
    sp = torch.cuda.current_stream().cuda_stream
    for i in range(6):
        check_engine(lib.msw_linear_decode(2, ws[i % copies].data_ptr(), ss[i % copies].data_ptr(), n, k,
                                           x.data_ptr(), 1, y.data_ptr(), sp))
    torch.cuda.synchronize()
    assert lib.msw_trace_set(C.c_void_p(buf.data_ptr())) == 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    check_engine(lib.msw_linear_decode(2, ws[0].data_ptr(), ss[0].data_ptr(), n, k, x.data_ptr(), 1,
                                       y.data_ptr(), sp))
    e1.record()
    torch.cuda.synchronize()
    lib.msw_trace_set(C.c_void_p(0))
    t = buf.cpu().numpy().reshape(148, 16).astype(np.int64)
    live = t[:, 14] != 0
    rel = (t[live, :10] - t[live, 14:15]) / 1965.0  # us
    g0 = t[live, 15]
    print(f"== W4 {name} n={n} k={k} ({wb / 1e6:.1f} MB) event {e0.elapsed_time(e1) * 1000:.2f} us, "
          f"{live.sum()} CTAs, start skew {(g0.max() - g0.min()) / 1000:.2f} us")
    for j, nm in enumerate(NAMES):
        col = rel[:, j]
        col = col[t[live, j] != 0]
        if len(col):
            print(f"  {j} {nm:13s} median {np.median(col):7.2f}  max {col.max():7.2f}  min {col.min():7.2f}")
