"""Profiling helper: one INT8 + continuous-batching cohort on the 8B shape."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2605_23057_b200 import MODE_INT8_CB, engine_cfg  # noqa: E402
from paper_2605_23057_b200.engine import Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=64)
ap.add_argument("--prompt", type=int, default=256)
ap.add_argument("--new", type=int, default=8)
a = ap.parse_args()
eng = Engine(engine_cfg(target="llama8b", draft=None, modes=[11], kv_blocks=a.n * ((a.prompt + a.new + 47) // 16) + 64, max_batch=64,
                        max_seq_len=a.prompt + a.new + 32))
rng = np.random.default_rng(0)
prompts = [rng.integers(0, eng.vocab, size=a.prompt).astype(np.int32) for _ in range(a.n)]
res = eng.run_batch(MODE_INT8_CB, prompts, [a.new] * a.n)
print("mean request ms", np.mean([r.total_ms for r in res]), "prefill ms", np.mean([r.prefill_ms for r in res]))
eng.close()
