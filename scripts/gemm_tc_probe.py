"""Runs the tcgen05 prefill/verify GEMM (gemm_tc_kernel, through msw_linear
with T > 6 tokens) on 8B shapes, for ncu captures of its tensor-pipe
utilisation: python scripts/gemm_tc_probe.py FMT N K T [reps]
(FMT 0 FP16, 1 INT8 W8A8, 2 W4 g128). Prints the CUDA-event time per launch
and the achieved dense TFLOP/s (2*N*K*T per launch)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_23057_b200._capi import check_engine, engine_lib  # noqa: E402

fmt, n, k, t = (int(a) for a in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 5
lib = engine_lib()
w16 = torch.empty((n, k), dtype=torch.int16, device="cuda")
check_engine(lib.msw_fill_fp16(w16.data_ptr(), n, k, 7, 4242, 6, None))
if fmt == 0:
    w, s = w16, None
elif fmt == 1:
    w = torch.empty((n, k), dtype=torch.int8, device="cuda")
    s = torch.empty(n, dtype=torch.float32, device="cuda")
    check_engine(lib.msw_quant_int8_rows(w16.data_ptr(), n, k, w.data_ptr(), s.data_ptr(), None))
else:
    w = torch.empty((n, k // 8), dtype=torch.int32, device="cuda")
    s = torch.empty((n, k // 128), dtype=torch.int16, device="cuda")
    check_engine(lib.msw_quant_w4_rows(w16.data_ptr(), n, k, w.data_ptr(), s.data_ptr(), None))
x = torch.randn((t, k), device="cuda")
y = torch.empty((t, n), device="cuda")
sp = torch.cuda.current_stream().cuda_stream


def go():
    check_engine(lib.msw_linear(fmt, w.data_ptr(), s.data_ptr() if s is not None else None, n, k,
                                x.data_ptr(), t, y.data_ptr(), sp))


for _ in range(2):
    go()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    go()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"fmt={fmt} n={n} k={k} T={t}: {ms * 1e3:.1f} us per msw_linear (prep + GEMM), "
      f"{2 * n * k * t / (ms * 1e-3) / 1e12:.1f} TFLOP/s", flush=True)
