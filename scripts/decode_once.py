"""Profiling helper: build the 8B-shape engine with one mode resident and run
one request (prompt P -> N new tokens) through the C ABI. Used under ncu."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2605_23057_b200 import engine_cfg  # noqa: E402
from paper_2605_23057_b200.engine import Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mode", type=int, default=2)
ap.add_argument("--prompt", type=int, default=128)
ap.add_argument("--new", type=int, default=4)
ap.add_argument("--target", default="llama8b")
ap.add_argument("--graphs", type=int, default=1)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
modes = [a.mode] if a.mode != 4 else [0, 4]
eng = Engine(engine_cfg(target=a.target, draft="llama1b" if a.mode == 4 else None, modes=modes,
                        kv_blocks=max(128, (a.prompt + a.new + 64) // 16 + 8), max_seq_len=a.prompt + a.new + 32, use_graphs=bool(a.graphs)))
p = np.random.default_rng(0).integers(0, eng.vocab, size=a.prompt).astype(np.int32)
for rep in range(a.reps):
    r = eng.run(a.mode, p, a.new)
    print("tokens", r.tokens[:4], "decode_ms", round(r.decode_ms, 3), "per_token_ms",
          round(r.decode_ms / max(1, a.new - 1), 4), "prefill_ms", round(r.prefill_ms, 3),
          "launches", r.kernel_launches, flush=True)
eng.close()
