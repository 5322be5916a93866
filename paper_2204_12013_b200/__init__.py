"""B200-native Bamboo redundant-computation pipeline (arXiv 2204.12013).

The product is the C-ABI library `libbamboo.so` (include/bamboo.h) with
hand-written sm_100a kernels and its own CUDA-IPC transport; this package is its thin ctypes
binding. Importing it loads the library and fails loudly if it is missing.
"""
from ._lib import (BambooError, Pipeline, session_id, plan_dump, lib, RC, xport_pingpong,  # noqa: F401
                   BB_E_UNSUPPORTED, BB_E_INVAL, BB_E_FATAL, BB_E_STATE,
                   op_gemm, op_attention_fwd, op_attention_bwd, op_layernorm_fwd,
                   op_layernorm_bwd, op_cross_entropy, op_adam, EXPORTED, LIB_PATH)

lib()
