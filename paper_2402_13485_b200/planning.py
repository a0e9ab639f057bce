"""Host side of dynamic tree generation (the scalar controller around K4).

The per-sequence statistics update and the node scoring/selection run on
the device (`propd_stats_replay_select`, acceptance.py:96-206).  What stays
here is the per-step controller the reference runs once per iteration:
the iteration-time model (cost_model.py:26-118), the size choice
(scheduler.py:41-69) and the replan triggers (scheduler.py:72-77,
engine.py:340-356) — a handful of fp64 scalars, plus `HeadPredictions`, the
return type of `draft` (acceptance.py:20-57).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


class HeadPredictions:
    """Per-head top-k drafts: tokens[d-1, r-1] is head d's rank-r token."""

    def __init__(self, tokens, scores) -> None:
        tokens = np.asarray(tokens, dtype=np.int64)
        scores = np.asarray(scores, dtype=np.float64)
        if tokens.ndim != 2 or tokens.shape != scores.shape:
            raise ValueError("tokens and scores must be matching 2-D arrays")
        for d in range(tokens.shape[0]):
            if np.unique(tokens[d]).size != tokens.shape[1]:
                raise ValueError(f"head {d + 1}: duplicate tokens in the top-k list")
        if np.any(np.diff(scores, axis=1) > 0):
            raise ValueError("scores must be non-increasing within each head")
        self.tokens, self.scores = tokens, scores

    @property
    def depth_count(self) -> int:
        return self.tokens.shape[0]

    @property
    def k_max(self) -> int:
        return self.tokens.shape[1]

    def token(self, depth: int, rank: int) -> int:
        if not (1 <= depth <= self.depth_count and 1 <= rank <= self.k_max):
            raise IndexError(f"no prediction at depth {depth}, rank {rank}")
        return int(self.tokens[depth - 1, rank - 1])

    def rank_of(self, depth: int, token: int):
        where = np.nonzero(self.tokens[depth - 1] == token)[0]
        return int(where[0]) + 1 if where.size else None


def grid_candidates(depth_count: int, k_max: int) -> tuple:
    """The selection universe: rank path (1,...,1,r) for every head d and rank r
    (acceptance.py:158-169).  Candidate index c = (d-1)*k_max + (r-1)."""
    return tuple((1,) * d + (r,) for d in range(depth_count) for r in range(1, k_max + 1))


def prewarm_P(depth_count: int, k_max: int) -> np.ndarray:
    """Initial cumulative hit curves min(0.9, 0.5^d) * r/k (acceptance.py:81-84)."""
    cap = np.minimum(0.9, 0.5 ** np.arange(1, depth_count + 1))
    return np.outer(cap, np.arange(1, k_max + 1) / k_max)


class InsufficientDataError(RuntimeError):
    """Fewer than two distinct sizes carry usable observations."""


class CostModel:
    """Per-size EMA of iteration time + staleness-weighted least-squares line."""

    def __init__(self, sizes, alpha: float = 0.2, staleness_decay: float = 0.01, prewarm_beta=None) -> None:
        uniq = sorted({int(s) for s in sizes})
        if not uniq or uniq[0] < 1:
            raise ValueError("sizes must be positive integers")
        if not 0.0 < alpha <= 1.0:
            raise ValueError("alpha must lie in (0, 1]")
        if staleness_decay < 0.0:
            raise ValueError("staleness_decay must be non-negative")
        self.sizes, self.alpha, self.staleness_decay = uniq, alpha, staleness_decay
        self._avg: dict = {}
        self._seen: dict = {}
        self._beta = None if prewarm_beta is None else (float(prewarm_beta[0]), float(prewarm_beta[1]))

    @property
    def beta(self):
        return self._beta

    def observe(self, size: int, t: float, now: int) -> None:
        if size not in self.sizes:
            raise ValueError(f"size {size} is not a tracked candidate")
        if not t > 0.0:
            raise ValueError("iteration time must be positive")
        old = self._avg.get(size)
        self._avg[size] = float(t) if old is None else (1.0 - self.alpha) * old + self.alpha * float(t)
        self._seen[size] = int(now)

    def weights(self, now: int) -> np.ndarray:
        return np.array([math.exp(-self.staleness_decay * (int(now) - self._seen[s])) if s in self._seen else 0.0
                         for s in self.sizes])

    def fit(self, now: int):
        w = self.weights(now)
        use = w > 0.0
        x = np.asarray(self.sizes, dtype=np.float64)[use]
        if np.unique(x).size < 2:
            raise InsufficientDataError("need observations at two distinct sizes to fit a line")
        y = np.array([self._avg[s] for s, u in zip(self.sizes, use) if u])
        w = w[use]
        sw = w.sum()
        sx, sy = float(w @ x), float(w @ y)
        sxx, sxy = float(w @ (x * x)), float(w @ (x * y))
        den = sw * sxx - sx * sx
        if den <= 0.0:
            raise InsufficientDataError("degenerate design: distinct sizes collapsed")
        slope = (sw * sxy - sx * sy) / den
        self._beta = ((sy - slope * sx) / sw, slope)
        return self._beta

    def estimate(self, size: int) -> float:
        if self._beta is None:
            raise InsufficientDataError("no fit has succeeded and no pre-warm line is set")
        return self._beta[0] + self._beta[1] * float(size)

    def reset(self) -> None:
        self._avg.clear()
        self._seen.clear()

    def diagnostics(self, now: int) -> list:
        w = self.weights(now)
        return [{"size": s, "t_perf": self._avg.get(s),
                 "staleness": None if s not in self._seen else int(now) - self._seen[s], "weight": float(wi)}
                for s, wi in zip(self.sizes, w)]


def choose_size(l_curve: dict, cost: CostModel, include_bonus: bool = False) -> int:
    """Best (l + bonus) / T_est over an ascending scan; ties keep the smaller
    size; an unusable estimate ends the scan; fallback = smallest size."""
    if not l_curve:
        raise ValueError("l_curve is empty")
    best, best_v = None, None
    extra = 1.0 if include_bonus else 0.0
    for size in sorted(l_curve):
        try:
            t = cost.estimate(size)
        except InsufficientDataError:
            break
        if t <= 0.0:
            continue
        v = (l_curve[size] + extra) / t
        if best_v is None or v > best_v:
            best, best_v = size, v
    return min(l_curve) if best is None else best


@dataclass(frozen=True)
class RuntimeSnapshot:
    batch: int
    mean_seqlen: float
    iterations_since_plan: int
    planned_batch: int
    planned_seqlen: float


def should_replan(snap: RuntimeSnapshot, cfg) -> bool:
    return (abs(snap.batch - snap.planned_batch) >= cfg.resize_batch_delta
            or abs(snap.mean_seqlen - snap.planned_seqlen) >= cfg.resize_seqlen_delta
            or snap.iterations_since_plan >= cfg.replan_period)


class LatencyModel:
    """Seeded simulated iteration clock (backends.py:568-603): the engine's
    time source for reproducible tree sizing in parity runs,
    t = c0_base + c0_batch B + c0_seqlen S + (c1_base + c1_batch B) rows
    + U(-noise, noise)."""

    def __init__(self, c0_base: float = 1.0, c0_batch: float = 0.0, c0_seqlen: float = 0.0, c1_base: float = 0.05,
                 c1_batch: float = 0.0, noise: float = 0.0, seed: int = 0) -> None:
        if noise < 0.0:
            raise ValueError("noise amplitude must be non-negative")
        self.c0 = (float(c0_base), float(c0_batch), float(c0_seqlen))
        self.c1 = (float(c1_base), float(c1_batch))
        self.noise = float(noise)
        self._rng = np.random.default_rng(seed)

    def iteration_time(self, rows: float, batch: int = 1, seqlen: float = 0.0) -> float:
        t = (self.c0[0] + self.c0[1] * batch + self.c0[2] * seqlen) + (self.c1[0] + self.c1[1] * batch) * float(rows)
        if self.noise > 0.0:
            t += float(self._rng.uniform(-self.noise, self.noise))
        if t <= 0.0:
            raise ValueError("latency coefficients produced a non-positive time")
        return float(t)
