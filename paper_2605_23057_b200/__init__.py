"""modeswitch-b200: B200-native executor for the inference modes routed by
ModeSwitch-LLM's request-boundary controller (arXiv 2605.23057).

Host controller (C++, libmodeswitch.so) + sm_100a CUDA engine
(libmsw_engine.so) behind C ABIs in include/. This package is the Python
handle over both; see DESIGN.md.
"""
from .configs import (ALL_MODES, MODE_AWQ4, MODE_CHUNKED_PREFILL, MODE_CUDA_GRAPHS, MODE_KV_COMPRESSION, MODE_FP16, MODE_GPTQ4,
                      MODE_GPTQ_PC, MODE_INT8, MODE_INT8_CB, MODE_NAMES, MODE_SPEC, ROUTED_MODES,
                      SCREENING_MODES, SHAPES, engine_cfg, model_cfg)

__all__ = ["ALL_MODES", "MODE_AWQ4", "MODE_CHUNKED_PREFILL", "MODE_CUDA_GRAPHS", "MODE_KV_COMPRESSION", "MODE_FP16", "MODE_GPTQ4",
           "MODE_GPTQ_PC", "MODE_INT8", "MODE_INT8_CB", "MODE_NAMES", "MODE_SPEC", "ROUTED_MODES",
           "SCREENING_MODES", "SHAPES", "engine_cfg", "model_cfg"]
