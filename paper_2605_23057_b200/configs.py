"""Model shapes (Llama-3.1-8B, Llama-3.2-1B-shape draft, and the builder's tiny
test model) and engine configurations. Random-init weights (K16), no
checkpoints: see DESIGN.md "Deterministic init"."""
from __future__ import annotations

from ._capi import EngineCfg, ModelCfg

LLAMA3_ROPE = dict(rms_eps=1e-5, rope_theta=500000.0, rope_factor=8.0,
                   rope_low_freq_factor=1.0, rope_high_freq_factor=4.0, rope_orig_ctx=8192)

SHAPES = {
    # Llama-3.1-8B: h 4096, 32 layers, 32 q / 8 kv heads of 128, FFN 14336, vocab 128256
    "llama8b": dict(hidden=4096, n_layers=32, n_heads=32, n_kv_heads=8, head_dim=128,
                    ffn=14336, vocab=128256, **LLAMA3_ROPE),
    # Llama-3.2-1B shape (draft): h 2048, 16 layers, 32/8 heads of 64, FFN 8192
    "llama1b": dict(hidden=2048, n_layers=16, n_heads=32, n_kv_heads=8, head_dim=64,
                    ffn=8192, vocab=128256, **LLAMA3_ROPE),
    # builder-defined tiny test model (SURVEY §8 suggested shape)
    "tiny": dict(hidden=512, n_layers=2, n_heads=8, n_kv_heads=2, head_dim=64,
                 ffn=1536, vocab=2048, **LLAMA3_ROPE),
    "tiny_draft": dict(hidden=256, n_layers=1, n_heads=4, n_kv_heads=2, head_dim=64,
                       ffn=768, vocab=2048, **LLAMA3_ROPE),
    # head_dim 128 variant of the tiny model (exercises the 8B attention path)
    "tiny128": dict(hidden=512, n_layers=2, n_heads=4, n_kv_heads=2, head_dim=128,
                    ffn=1536, vocab=2048, **LLAMA3_ROPE),
}

MODE_FP16, MODE_INT8, MODE_GPTQ4, MODE_SPEC, MODE_GPTQ_PC, MODE_INT8_CB = 0, 1, 2, 4, 10, 11
MODE_AWQ4, MODE_CHUNKED_PREFILL, MODE_CUDA_GRAPHS, MODE_KV_COMPRESSION = 3, 6, 8, 9  # screening (not routed)
ROUTED_MODES = (MODE_FP16, MODE_INT8, MODE_GPTQ4, MODE_SPEC, MODE_GPTQ_PC, MODE_INT8_CB)
SCREENING_MODES = (MODE_AWQ4, MODE_CHUNKED_PREFILL, MODE_CUDA_GRAPHS, MODE_KV_COMPRESSION)
ALL_MODES = ROUTED_MODES + SCREENING_MODES
MODE_NAMES = {0: "fp16", 1: "int8", 2: "gptq4", 3: "awq4", 4: "speculative_decoding", 6: "chunked_prefill",
              8: "cuda_graphs", 9: "kv_cache_compression", 10: "gptq_prefix_caching", 11: "int8_continuous_batching"}


def model_cfg(name: str) -> ModelCfg:
    return ModelCfg(**SHAPES[name])


def modes_mask(modes=ALL_MODES) -> int:
    m = 0
    for x in modes:
        m |= 1 << x
    return m


def engine_cfg(target: str = "tiny", draft: str | None = "tiny_draft", modes=ALL_MODES,
               seed: int = 0, agree_permille: int = 800, kv_blocks: int = 4096,
               max_batch: int = 64, max_seq_len: int = 2048, spec_k: int = 4,
               use_graphs: bool = True) -> EngineCfg:
    cfg = EngineCfg()
    cfg.target = model_cfg(target)
    if draft is not None:
        cfg.draft = model_cfg(draft)
        cfg.has_draft = 1
    cfg.modes_mask = modes_mask(modes)
    cfg.weight_seed = seed
    cfg.draft_agree_permille = agree_permille
    cfg.kv_blocks = kv_blocks
    cfg.max_batch = max_batch
    cfg.max_seq_len = max_seq_len
    cfg.spec_k = spec_k
    cfg.use_graphs = int(use_graphs)
    return cfg
