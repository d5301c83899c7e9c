"""Kernel-only timing of the tcgen05 prefill GEMM through the engine's own
linear path: msw_linear repacks weights per call, so instead this builds the
8B engine once and times its packed prefill (prefill_ms, CUDA events) at
several prompt lengths per mode. Usage: gemm_tc_time.py [T ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2605_23057_b200 import engine_cfg  # noqa: E402
from paper_2605_23057_b200.configs import model_cfg  # noqa: E402
from paper_2605_23057_b200.engine import Engine  # noqa: E402

lens = [int(a) for a in sys.argv[1:]] or [128, 1024, 2048]
eng = Engine(engine_cfg(target="llama8b", draft=None, modes=[0, 1, 2], kv_blocks=1024,
                        max_seq_len=max(lens) + 64, use_graphs=True))
c = model_cfg("llama8b")
lin = 2 * (c.n_layers * (c.hidden * (c.n_heads + 2 * c.n_kv_heads) * c.head_dim +
                         c.n_heads * c.head_dim * c.hidden + 3 * c.hidden * c.ffn) + c.vocab * c.hidden)
for T in lens:
    p = np.random.default_rng(T).integers(0, c.vocab, size=T).astype(np.int32)
    for mode, name in ((0, "fp16"), (1, "int8"), (2, "gptq4")):
        eng.run(mode, p, 2)
        ms = min(eng.run(mode, p, 2).prefill_ms for _ in range(3))
        att = 4.0 * c.n_layers * c.n_heads * c.head_dim * T * (T + 1) / 2
        print(f"T={T:5d} {name:6s} prefill {ms:8.2f} ms  {(lin * T / 2 * 2 + att) / (ms * 1e-3) / 1e12:6.1f} "
              f"TFLOP/s (linears + causal attention)", flush=True)
eng.close()
