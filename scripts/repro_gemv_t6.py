"""Stress the FP16 6-token decode GEMV at K = 14336 (2-stage ring, 168 KB
activation stage): compare each run against the first (bitwise; the kernel is
deterministic) and against the oracle; report mismatching runs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
from paper_2605_23057_b200 import _capi  # noqa: E402
from paper_2605_23057_b200._capi import check_engine, engine_lib  # noqa: E402

n, k = int(sys.argv[1]) if len(sys.argv) > 1 else 256, 14336
t = int(sys.argv[3]) if len(sys.argv) > 3 else 6
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 300
rng = np.random.default_rng(t * 1000 + n)
w = O.fill_fp16(n, k, 11, 1234 + n, (int(np.ceil(np.log2(k))) + 1) // 2)
x = rng.standard_normal((t, k)).astype(np.float32)
x[:, 0] = 4.0
ref = O.linear(_capi.W_FP16, w, None, x)
dw = torch.from_numpy(w.view(np.int16)).cuda()
dx = torch.from_numpy(x).cuda()
first, bad = None, 0
for i in range(iters):
    dy = torch.empty((t, n), dtype=torch.float32, device="cuda")
    check_engine(engine_lib().msw_linear(_capi.W_FP16, dw.data_ptr(), None, n, k, dx.data_ptr(), t,
                                         dy.data_ptr(), None))
    torch.cuda.synchronize()
    y = dy.cpu().numpy()
    err = np.abs(y - ref).max() / np.abs(ref).max()
    if first is None:
        first = y
    if err >= 2e-5 or not np.array_equal(y, first):
        bad += 1
        idx = np.unravel_index(np.argmax(np.abs(y - ref)), y.shape)
        print(f"run {i}: rel err {err:.3g} at token {idx[0]} row {idx[1]}, "
              f"bitwise-diff elems {int((y != first).sum())}", flush=True)
print(f"n={n} t={t}: {bad} bad of {iters}")
