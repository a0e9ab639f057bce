"""B200-native batched ProPD token-tree decode step (arXiv 2402.13485).

Drop-in for the reference package `treedecode`'s hot path: `B200Backend`
implements its ModelBackend plugin API (backends.py:53-95) on hand-written
sm_100a kernels (libpropd.so, C ABI in include/propd.h), and `DecodeEngine`
is the batched decode loop with the reference's run()/metrics surface
(engine.py:139-414).
"""

from .config import (MODES, VICUNA_7B_SHAPE, VICUNA_33B_SHAPE, EngineConfig, PruneConfig, SchedulerConfig,
                     TinyTransformerConfig)
from .planning import CostModel, HeadPredictions, InsufficientDataError, LatencyModel, choose_size, grid_candidates
from .tree import TreeTemplate

__all__ = [
    "MODES", "VICUNA_7B_SHAPE", "VICUNA_33B_SHAPE", "EngineConfig", "PruneConfig", "SchedulerConfig",
    "TinyTransformerConfig", "CostModel", "HeadPredictions", "InsufficientDataError", "LatencyModel", "choose_size",
    "grid_candidates", "TreeTemplate", "B200Backend", "DecodeEngine",
]


def __getattr__(name):
    # torch-dependent pieces load lazily so the CPU-only tests import cheaply
    if name in ("B200Backend", "DecodeState", "TreeForward"):
        from . import backend

        return getattr(backend, name)
    if name in ("DecodeEngine", "RunResult", "IterationMetrics"):
        from . import engine

        return getattr(engine, name)
    raise AttributeError(name)
