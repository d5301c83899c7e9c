"""Prefill / decode-step kernel attribution on the 8B shape: run under
`ncu --metrics gpu__time_duration.sum --csv` and summarise with
scripts/ncu_sum.py. One request per mode: prompt P, 2 new tokens (eager)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_23057_b200 import MODE_FP16, MODE_GPTQ4, MODE_INT8, engine_cfg  # noqa: E402
from paper_2605_23057_b200.engine import Engine  # noqa: E402

P = int(os.environ.get("P", "128"))
modes = [int(m) for m in os.environ.get("MODES", "0,1,2").split(",")]
eng = Engine(engine_cfg(target="llama8b", draft=None, modes=modes, seed=0, kv_blocks=1024,
                        max_seq_len=max(512, P + 64), use_graphs=False))
p = (np.arange(P, dtype=np.int64) * 7919 % 128256).astype(np.int32)
for m in modes:
    eng.run(m, p, 2)  # warm (attrs, tensor maps)
for m in modes:
    r = eng.run(m, p, 2)
    print(f"mode {m}: prefill_ms {r.prefill_ms:.3f} total_ms {r.total_ms:.3f}", flush=True)
eng.close()
