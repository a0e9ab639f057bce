"""Configuration records with the reference's field names, defaults and
validation messages, so reference-style code constructs them unchanged.

Mirrors (paths relative to /root/reference/pkg/src/treedecode/):
  TinyTransformerConfig  backends.py:116-132
  PruneConfig            pruning.py:22-30
  SchedulerConfig        scheduler.py:20-31
  EngineConfig / MODES   engine.py:28-66
"""

from __future__ import annotations

from dataclasses import dataclass

RankPath = tuple  # tuple[int, ...]: per-head ranks along a root-to-node path

MODES = ("autoregressive", "static_tree", "prune_only", "dynamic_only", "propd_full")


@dataclass(frozen=True)
class TinyTransformerConfig:
    """Model shape + seed.  The 7B shape is layers=32, hidden=4096, heads=32,
    vocab=32000 (the transformer block is the reference's pre-LN GPT-2 style)."""

    layers: int = 4
    hidden: int = 64
    heads: int = 4
    vocab: int = 256
    draft_heads: int = 4
    max_positions: int = 512
    seed: int = 0

    def __post_init__(self) -> None:
        if self.layers < 1 or self.hidden < 1 or self.heads < 1:
            raise ValueError("layers, hidden, and heads must be positive")
        if self.hidden % self.heads != 0:
            raise ValueError("hidden must be divisible by heads")
        if self.vocab < 2 or self.draft_heads < 1 or self.max_positions < 2:
            raise ValueError("vocab, draft_heads, max_positions too small")

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads


VICUNA_7B_SHAPE = dict(layers=32, hidden=4096, heads=32, vocab=32000, draft_heads=4)
VICUNA_33B_SHAPE = dict(layers=60, hidden=6656, heads=52, vocab=32000, draft_heads=4)


@dataclass(frozen=True)
class PruneConfig:
    """Top-K early pruning (pruning.py:22-30, 40-66); with `threshold` set,
    probability-based pruning instead: a node survives iff its marginal path
    probability under the early head is >= threshold (the
    reference disables this criterion, pruning.py:76-82)."""

    layer: int = 4
    topk: int = 50
    threshold: float | None = None

    def __post_init__(self) -> None:
        if self.layer < 1:
            raise ValueError("prune layer must be >= 1")
        if self.topk < 1:
            raise ValueError("prune top-K must be >= 1")
        if self.threshold is not None and not 0.0 < self.threshold <= 1.0:
            raise ValueError("prune threshold must lie in (0, 1]")


@dataclass(frozen=True)
class SchedulerConfig:
    resize_batch_delta: int = 1
    resize_seqlen_delta: int = 256
    replan_period: int = 16
    size_candidates: tuple = (1, 2, 4, 8, 16, 32, 64)

    def __post_init__(self) -> None:
        if self.resize_batch_delta < 1 or self.resize_seqlen_delta < 1 or self.replan_period < 1:
            raise ValueError("replan thresholds must be positive")
        if not self.size_candidates or any(s < 1 for s in self.size_candidates):
            raise ValueError("size candidates must be positive")


@dataclass(frozen=True)
class EngineConfig:
    mode: str = "propd_full"
    draft_heads: int = 4
    draft_topk: int = 3
    prune: PruneConfig | None = None
    scheduler: SchedulerConfig = SchedulerConfig()
    static_tree: tuple | None = None
    acceptance_alpha: float | None = 0.05
    cost_alpha: float = 0.2
    cost_staleness: float = 0.01
    include_bonus_in_speed: bool = False
    probe_rounds: int = 1
    eos_token: int | None = None
    # "greedy" (verification.py:30-53) or "typical": candidate x accepted iff
    # log p(x) > min(log epsilon, log alpha - H(p)), p = softmax(logits / T)
    acceptance: str = "greedy"
    typical_epsilon: float = 0.09
    typical_alpha: float = 0.3
    typical_temperature: float = 1.0

    def __post_init__(self) -> None:
        if self.acceptance not in ("greedy", "typical"):
            raise ValueError("acceptance must be 'greedy' or 'typical'")
        if not (self.typical_epsilon > 0 and self.typical_alpha > 0 and self.typical_temperature > 0):
            raise ValueError("typical acceptance parameters must be positive")
        if self.mode not in MODES:
            raise ValueError(f"unknown mode {self.mode!r}; expected one of {MODES}")
        if self.draft_heads < 1 or self.draft_topk < 1:
            raise ValueError("draft_heads and draft_topk must be positive")
        if self.uses_prune and self.prune is None:
            raise ValueError(f"mode {self.mode!r} needs a prune config")
        if self.probe_rounds < 0:
            raise ValueError("probe_rounds must be non-negative")

    @property
    def uses_tree(self) -> bool:
        return self.mode != "autoregressive"

    @property
    def uses_prune(self) -> bool:
        return self.mode in ("prune_only", "propd_full")

    @property
    def uses_dynamic(self) -> bool:
        return self.mode in ("dynamic_only", "propd_full")
