"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NO arithmetic of the method (no model op, no schedule,
no RC/recovery rule). It only defines the workload shapes
and draws the seeded token ids and initial weights (SURVEY.md §8(d),
"Synthetic inputs"). Both `oracle/` and the product binding's callers
(tests, bench.py) import it; neither side imports the other.
"""
from .configs import ModelCfg, RunCfg, CONFIGS, get_config, depth_reduced  # noqa: F401
from .inputs import make_tokens, make_params, param_specs, n_params, round_to_bf16  # noqa: F401
