"""Workload shapes (BASELINE.json `configs`).

Model dimensions follow the paper's benchmark models (PAPER.md P:630-631,
"BERT-Large", "GPT-2"); the values marked † in SURVEY.md §8.0 (padded vocab,
micro-batch size) are this build's readings, listed in DESIGN.md.
"""
from dataclasses import dataclass, replace


@dataclass(frozen=True)
class ModelCfg:
    n_layer: int
    d_model: int
    n_head: int
    d_ff: int
    vocab: int            # padded vocab, used everywhere (embedding + head rows)
    vocab_sample: int     # token ids are drawn below this (unpadded size)
    seq_len: int
    causal: bool

    @property
    def d_head(self) -> int:
        return self.d_model // self.n_head


@dataclass(frozen=True)
class RunCfg:
    name: str
    index: int            # config index in BASELINE.json (seeds tokens)
    model: ModelCfg
    stages: int           # P
    microbatches: int     # M
    micro_batch: int      # mb (sequences per micro-batch)
    gpt: bool             # GPT (shifted targets) vs BERT (independent targets)

    @property
    def samples_per_step(self) -> int:
        return self.microbatches * self.micro_batch


CONFIGS = {
    "C0": RunCfg("C0", 0, ModelCfg(4, 64, 2, 256, 128, 128, 32, True), 2, 4, 2, True),
    "C1": RunCfg("C1", 1, ModelCfg(12, 768, 12, 3072, 50304, 50257, 1024, True), 4, 8, 8, True),
    "C2": RunCfg("C2", 2, ModelCfg(24, 1024, 16, 4096, 30528, 30522, 512, False), 8, 16, 16, False),
    "C3": RunCfg("C3", 3, ModelCfg(48, 1600, 25, 6400, 50304, 50257, 1024, True), 8, 32, 4, True),
}


def get_config(name: str) -> RunCfg:
    return CONFIGS[name]


def depth_reduced(name: str, blocks_per_stage: int = 1, microbatches: int = 4,
                  micro_batch: int | None = None) -> RunCfg:
    """Width-exact, depth-reduced variant (SURVEY.md §8(c) parity tier PT2)."""
    c = CONFIGS[name]
    m = replace(c.model, n_layer=blocks_per_stage * c.stages)
    return replace(c, name=f"{name}-d{blocks_per_stage}", model=m, microbatches=microbatches,
                   micro_batch=c.micro_batch if micro_batch is None else micro_batch)
