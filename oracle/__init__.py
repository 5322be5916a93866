"""Bamboo oracle — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct fp64 CPU implementation (numpy) of what the
hot path computes: the GPT/BERT-style transformer (model.py), the pipeline
partition and 1F1B + eager-FRC plans (plan.py), and the plan interpreter with
redundant-computation, preemption-injection and recovery semantics
(pipeline.py), each following PAPER.md (arXiv 2204.12013) as cited.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs may import this package. The product path
(`paper_2204_12013_b200/`, `include/`, the CUDA library) never imports,
links or calls it, and shares no code with it; only the seeded input
generators in `synth/` serve both.

Parity status: every function is pinned by a `-m "not gpu"` test in
tests/test_oracle_*.py (finite differences, torch library routines,
closed forms, paper examples, brute force). None is "parity unpinned".
"""
