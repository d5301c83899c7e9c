"""In-graph timeline of the split-KV decode attention kernel (diagnostics
build, -DMSW_TRACE): globaltimer per CTA at entry (0), past griddepcontrol.wait
(1), RoPE done (2), positions done (3), partial written (4), merge done (5,
last split only), idle-split exit (7); reported for the last attention launch
of the run (last layer of the last decode step), relative to the first entry."""
import ctypes as C
import os
import sys

os.environ.setdefault("MSW_ENGINE_SO", "libmsw_engine_trace.so")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_23057_b200 import engine_cfg  # noqa: E402
from paper_2605_23057_b200._capi import engine_lib  # noqa: E402
from paper_2605_23057_b200.engine import Engine  # noqa: E402

mode = int(sys.argv[1]) if len(sys.argv) > 1 else 2
prompt = int(sys.argv[2]) if len(sys.argv) > 2 else 200
lib = engine_lib()
eng = Engine(engine_cfg(target="llama8b", draft=None, modes=[mode], kv_blocks=640, max_seq_len=prompt + 64))
p = np.arange(prompt, dtype=np.int32) % 1000
eng.run(mode, p, 4)
buf = torch.zeros(8 * 8 * 64 * 8, dtype=torch.int64, device="cuda")
assert lib.msw_attn_trace_set(C.c_void_p(buf.data_ptr())) == 0
eng.run(mode, p, 3)
torch.cuda.synchronize()
lib.msw_attn_trace_set(C.c_void_p(0))
t = buf.cpu().numpy().reshape(-1, 8)
live = t[:, 0] > 0
t = t[live]
t0 = t[:, 0].min()
print(f"ctx {prompt + 2}: {live.sum()} CTAs recorded")
for e, nm in enumerate(["entry", "past pdl wait", "rope done", "positions done", "partial written",
                        "merge|QK done", "tile 0 staged", "idle exit"]):
    col = t[:, e]
    col = col[col > 0]
    if len(col):
        r = (col - t0) / 1000.0
        print(f"  {e} {nm:16s} n={len(col):3d} min {r.min():7.2f} median {np.median(r):7.2f} max {r.max():7.2f} us")
eng.close()
