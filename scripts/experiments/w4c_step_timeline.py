"""In-step timeline of the two-CTA W4 decode GEMVs (diagnostics build of
gemv_w4.cu with -DMSW_TRACE, MSW_ENGINE_SO=libmsw_engine_w4ctr.so): decodes
an 8B-shape GPTQ4 request through the engine (CUDA-graph step) with the
globaltimer trace armed, then prints, per linear class (qkv, o, gate_up,
down: launch index mod 4), the median over the traced launches of
  gap   = this launch's first consumer past griddepcontrol.wait - the previous
          W4 launch's last epilogue done (attention / lm_head sit in between),
  pro   = first stage consumed - past PDL wait (prologue),
  body  = last consumer done - first stage consumed,
  tail  = last epilogue done - last consumer done,
and the SM-doubling count."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_23057_b200 import engine_cfg  # noqa: E402
from paper_2605_23057_b200._capi import engine_lib  # noqa: E402
from paper_2605_23057_b200.engine import Engine  # noqa: E402

eng = Engine(engine_cfg(target="llama8b", draft=None, modes=[2], kv_blocks=128, max_seq_len=300, use_graphs=True))
p = np.random.default_rng(0).integers(0, eng.vocab, size=128).astype(np.int32)
eng.run(2, p, 8)
lib = engine_lib()
tr = torch.zeros(512 * 148 * 8, dtype=torch.int64, device="cuda")
torch.cuda.synchronize()
assert lib.msw_w4c_trace_set(C.c_void_p(tr.data_ptr())) == 0
r = eng.run(2, p, 6)
torch.cuda.synchronize()
lib.msw_w4c_trace_set(C.c_void_p(0))
print("decode ms/token", r.decode_ms / 5)
t = tr.cpu().numpy().reshape(512, 148, 8).astype(np.int64)
nl = int((t[:, :, 1].max(axis=1) > 0).sum())
names = ["qkv", "o", "gate_up", "down"]
rows = {n: [] for n in names}
for L in range(1, nl):
    a, b = t[L - 1], t[L]
    la, lb = a[:, 1] > 0, b[:, 1] > 0
    gap = (b[lb, 2].min() - a[la, 5].max()) / 1e3
    pro = (np.median(b[lb, 3]) - np.median(b[lb, 2])) / 1e3
    body = (b[lb, 4].max() - np.median(b[lb, 3])) / 1e3
    tail = (b[lb, 5].max() - b[lb, 4].max()) / 1e3
    total = (b[lb, 5].max() - a[la, 5].max()) / 1e3
    uniq, cnt = np.unique(b[lb, 0], return_counts=True)
    rows[names[L % 4]].append((gap, pro, body, tail, total, int((cnt > 1).sum())))
print(f"{nl} W4 launches traced")
for n in names:
    a = np.array(rows[n])
    if len(a):
        m = np.median(a, axis=0)
        print(f"{n:8s} gap {m[0]:6.2f}  pro {m[1]:6.2f}  body {m[2]:6.2f}  tail {m[3]:6.2f}  "
              f"end-to-end {m[4]:6.2f} us  doubled SMs max {int(a[:, 5].max())}")
eng.close()
