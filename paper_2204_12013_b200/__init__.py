"""B200-native Bamboo redundant-computation pipeline (arXiv 2204.12013).

The product is the C-ABI library `libbamboo.so` (include/bamboo.h) with
hand-written sm_100a kernels and NCCL P2P; this package is its thin ctypes
binding. Importing it loads the library and fails loudly if it is missing.
"""
from ._lib import (BambooError, Pipeline, nccl_unique_id, plan_dump, lib,  # noqa: F401
                   op_gemm, op_attention_fwd, op_attention_bwd, op_layernorm_fwd,
                   op_layernorm_bwd, op_cross_entropy, op_adam, EXPORTED, LIB_PATH)

lib()
