"""Batched decode loop over the B200 backend.

Same public surface and per-iteration semantics as the reference
DecodeEngine (engine.py:139-414): `run(prompts, max_tokens, batch_size)`
returns transcripts, per-iteration metrics, plan events and a summary that
equal the reference's for the same model, prompts and simulated clock.

What changes is where the work happens.  The reference loops over sequences
in Python and calls draft / forward_tree / verify / commit / stats.update
one sequence at a time (engine.py:257-288); here one `step_tree` call runs
the whole batch on the device, and the acceptance statistics are replayed
on the device in batch order from integer acceptance records
(`propd_stats_replay_select`), which is exactly the reference's sequential
update order.  With a torch.distributed process group the batch is sharded
across ranks (one model replica per GPU); each step all-gathers the records
so every rank replays the same global sequence order and plans the same tree.
"""

from __future__ import annotations

import time
from collections import deque
from dataclasses import dataclass

import numpy as np

from .config import EngineConfig
from .parallel import COL_ACC, COL_FIN, COL_KEPT, COL_RANKS, COL_SURV, global_rows, record_width, step_exchange
from .planning import (CostModel, InsufficientDataError, RuntimeSnapshot, choose_size, grid_candidates,
                       prewarm_P, should_replan)
from .tree import TreeTemplate


@dataclass(frozen=True)
class IterationMetrics:
    iteration: int
    batch: int
    mean_seqlen: float
    tree_size: int
    mean_survivors: float
    prune_rate: float
    mean_accepted: float
    tokens_committed: int
    iteration_time: float
    replanned: bool

    def to_json(self) -> dict:
        return {k: getattr(self, k) for k in self.__dataclass_fields__}


@dataclass(frozen=True)
class PlanEvent:
    iteration: int
    trigger: str
    chosen_size: int
    l_curve: dict
    v_curve: dict


@dataclass(frozen=True)
class RunSummary:
    mode: str
    iterations: int
    total_tokens: int
    total_time: float
    tokens_per_sec: float
    mean_accepted: float
    mean_prune_rate: float
    mean_tree_size: float


@dataclass(frozen=True)
class RunResult:
    transcripts: list
    prompts: list
    metrics: list
    plan_events: list
    summary: RunSummary


class _Seq:
    __slots__ = ("state", "prompt", "generated", "finished", "gid")

    def __init__(self, state, prompt, gid):
        self.state, self.prompt, self.generated, self.finished, self.gid = state, prompt, [], False, gid


class DecodeEngine:
    """Batched ProPD decode loop; `latency_model` (any object with
    iteration_time(rows, batch=, seqlen=)) drives a simulated clock, else
    wall time with a device synchronisation per iteration."""

    def __init__(self, backend, config: EngineConfig, latency_model=None, *, group=None, trace=None) -> None:
        self.backend, self.config, self.latency = backend, config, latency_model
        self.trace = trace
        self.group = group
        if config.uses_tree:
            if config.draft_heads != backend.draft_head_count:
                raise ValueError("engine draft_heads must match the backend's head count")
            if config.draft_topk >= backend.vocab_size:
                raise ValueError("draft_topk must be smaller than the vocabulary")
            if config.draft_topk > 127:  # acceptance records: rank + 1 in an int8 (propd_stats_replay_select)
                raise ValueError("draft_topk above 127 is not supported by the device acceptance records")
        if config.uses_prune and not 1 <= config.prune.layer < backend.num_layers:
            raise ValueError("prune layer must lie strictly inside the backbone")
        D, k = config.draft_heads, config.draft_topk
        grid = D * k
        self.size_candidates = sorted({min(int(s), grid) for s in config.scheduler.size_candidates})
        self.universe = grid_candidates(D, k)
        if config.mode in ("static_tree", "prune_only"):
            self.static_paths = tuple(config.static_tree) if config.static_tree is not None else self.universe
        else:
            self.static_paths = ()
        sizes = set(self.size_candidates) | ({len(self.static_paths)} if self.static_paths else set())
        self.cost = CostModel(sizes, alpha=config.cost_alpha, staleness_decay=config.cost_staleness)
        _warm_host_math()
        self._templates: dict = {}
        self._iteration = 0
        self._selection = None
        self._planned_batch = None
        self._planned_seqlen = 0.0
        self._planned_iteration = 0
        self._probe_queue = deque(self.size_candidates * config.probe_rounds)
        self.plan_events: list = []
        # acceptance statistics live on the device (fp64), K4 replays into them
        import torch

        dev = backend.device
        self._P = torch.tensor(prewarm_P(D, k), dtype=torch.float64, device=dev)
        self._counts = torch.zeros(D, dtype=torch.int64, device=dev)
        self._order_dev = torch.empty(grid, dtype=torch.int32, device=dev)
        self._lcurve_dev = torch.empty(grid, dtype=torch.float64, device=dev)
        if config.uses_tree:
            empty = torch.zeros(1, D, dtype=torch.int8, device=dev)
            backend.stats_replay_select(empty, 0, self._P, self._counts, config.acceptance_alpha,
                                        self._order_dev, self._lcurve_dev)
            self._pull_selection()

    # ------------------------------------------------------------- stats
    @property
    def stats_P(self) -> np.ndarray:
        return self._P.cpu().numpy()

    def _pull_selection(self) -> None:
        self._order = self._order_dev.cpu().numpy()
        self._lcurve = self._lcurve_dev.cpu().numpy()

    def _select(self, sizes) -> dict:
        """{size: (paths, expected length)} from the device-computed order."""
        return {s: (tuple(self.universe[c] for c in self._order[:s]), float(self._lcurve[s - 1])) for s in sizes}

    def _template(self, paths) -> TreeTemplate:
        key = tuple(paths)
        t = self._templates.get(key)
        if t is None:
            t = TreeTemplate.from_paths(paths, self.config.draft_heads, self.config.draft_topk)
            self._templates[key] = t
        return t

    # ------------------------------------------------------------- run
    def run(self, prompts, max_tokens: int, batch_size: int | None = None) -> RunResult:
        if max_tokens < 1:
            raise ValueError("max_tokens must be positive")
        prompts = [list(map(int, p)) for p in prompts]
        if not prompts or any(len(p) == 0 for p in prompts):
            raise ValueError("prompts must be non-empty")
        chunk = len(prompts) if batch_size is None else max(1, int(batch_size))
        rank, world = self._rank_world()
        transcripts, metrics = [], []
        for lo in range(0, len(prompts), chunk):
            group = prompts[lo: lo + chunk]
            mine = _shard(len(group), rank, world)
            states = self.backend.prefill_batch([group[i] for i in mine]) if mine else []
            seqs = [_Seq(st, group[i], lo + i) for st, i in zip(states, mine)]
            active = list(seqs)
            # multi-rank: every rank tracks the whole chunk from the per-step tables
            self._glob = _Global(group, world) if self.group is not None else None
            while self._glob.any_active() if self._glob is not None else active:
                metrics.append(self._step(active, max_tokens))
                active = [s for s in seqs if not s.finished]
            transcripts.extend(self._glob.transcripts if self._glob is not None else [s.generated for s in seqs])
            self._glob = None
            for s in seqs:
                self.backend.release(s.state)
        return RunResult(transcripts, prompts, metrics, list(self.plan_events), self._summarize(metrics))

    # ------------------------------------------------------------- step
    def _step(self, active: list, max_tokens: int) -> IterationMetrics:
        self._iteration += 1
        glob = getattr(self, "_glob", None)
        if glob is not None:
            batch, mean_seqlen = glob.batch_stats()
        else:
            batch, mean_seqlen = len(active), float(np.mean([s.state.length for s in active]))
        wall0 = time.perf_counter() if self.latency is None else 0.0
        cfg = self.config
        D = cfg.draft_heads
        if not cfg.uses_tree:
            toks = self.backend.step_autoregressive([s.state for s in active]) if active else []
            kept = [self._absorb(s, [int(t)], max_tokens) for s, t in zip(active, toks)]
            if glob is None:
                committed = sum(kept)
                t = self._clock(wall0, 1.0, batch, mean_seqlen)
            else:
                rows = np.zeros((len(active), record_width(D)), dtype=np.int32)
                rows[:, COL_RANKS + D + 1:] = -1
                for i, (s, tk) in enumerate(zip(active, toks)):
                    rows[i, COL_KEPT], rows[i, COL_FIN], rows[i, COL_RANKS + D] = kept[i], int(s.finished), int(tk)
                hrows, t_wall = self._exchange(rows, wall0)
                committed = int(hrows[:, COL_KEPT].sum())
                t = self._clock(wall0, 1.0, batch, mean_seqlen, t_wall)
            return IterationMetrics(self._iteration, batch, mean_seqlen, 0, 0.0, 0.0, 0.0, committed, t, False)

        paths, replanned = self._plan(batch, mean_seqlen)
        tmpl = self._template(paths)
        n = len(tmpl)  # nodes of the built tree (prune rate denominator, pruning.py:65)
        drafted_n = len(paths)  # the reference's tree size: rows formula, cost.observe (engine.py:252, 290-298)
        prune = cfg.prune if cfg.uses_prune else None
        states = [s.state for s in active]
        stats = None
        if glob is None:  # single process: the backend replays the records in the step's batch
            stats = (self._P, self._counts, cfg.acceptance_alpha, self._order_dev, self._lcurve_dev)
        accept = ((cfg.typical_epsilon, cfg.typical_alpha, cfg.typical_temperature)
                  if cfg.acceptance == "typical" else None)
        out = self.backend.step_tree(states, tmpl, cfg.draft_topk, prune, trace=self.trace is not None,
                                     stats=stats, accept=accept) if active else None
        kept = []
        for i, s in enumerate(active):
            a = int(out.acc_len[i])
            kept.append(self._absorb(s, [int(t) for t in out.committed[i, : a + 1]], max_tokens))
            if self.trace is not None:
                self._emit_trace(s, i, out, tmpl, a)
        t_wall = None
        if glob is None:
            self._order, self._lcurve = out.order, out.lcurve
            acc = out.acc_len.astype(np.int64)
            surv = out.surv_cnt.astype(np.int64)
            committed = sum(kept)
        else:
            rows = np.zeros((len(active), record_width(D)), dtype=np.int32)
            if active:
                rows[:, COL_ACC], rows[:, COL_SURV] = out.acc_len, out.surv_cnt
                rows[:, COL_KEPT] = kept
                rows[:, COL_FIN] = [int(s.finished) for s in active]
                rows[:, COL_RANKS: COL_RANKS + D] = out.ranks
                rows[:, COL_RANKS + D:] = out.committed
            hrows, t_wall = self._exchange(rows, wall0)
            acc = hrows[:, COL_ACC].astype(np.int64)
            surv = hrows[:, COL_SURV].astype(np.int64)
            committed = int(hrows[:, COL_KEPT].sum())
            self._pull_selection()
        acc_total, surv_total = int(acc.sum()), int(surv.sum())
        surv_mean = surv_total / batch
        if prune is not None:
            p, Ly = prune.layer, self.backend.num_layers
            rows_eff = (p * drafted_n + (Ly - p) * surv_mean) / Ly
            rates = [1.0 - int(c) / n for c in surv]  # global sequence order
            prune_rate = float(np.mean(rates)) if rates else 0.0  # numpy's pairwise sum, as the reference
        else:
            rows_eff, prune_rate = float(drafted_n), 0.0
        t = self._clock(wall0, rows_eff, batch, mean_seqlen, t_wall)
        self.cost.observe(drafted_n, t, now=self._iteration)
        return IterationMetrics(self._iteration, batch, mean_seqlen, drafted_n, surv_mean, prune_rate,
                                acc_total / batch, committed, t, replanned)

    def _exchange(self, rows: np.ndarray, wall0: float):
        """The step's one collective: every rank's records in global order;
        replays the acceptance records into P (tree modes) and advances the
        chunk's global view.  Returns (rows [S, R], max step seconds or None)."""
        import torch

        glob, D = self._glob, self.config.draft_heads
        us = 0
        if self.latency is None:
            torch.cuda.synchronize(self.backend.device)
            us = int(min((time.perf_counter() - wall0) * 1e6, 2**31 - 1))
        table = step_exchange(rows, us, glob.cap, self.group)
        hrows, step_us, drows = global_rows(table)
        if self.config.uses_tree:
            ranks = drows[:, COL_RANKS: COL_RANKS + D].to(torch.int8).to(self.backend.device)
            if ranks.shape[0] == 0:
                ranks = torch.zeros(1, D, dtype=torch.int8, device=self.backend.device)
            self.backend.stats_replay_select(ranks, int(hrows.shape[0]), self._P, self._counts,
                                             self.config.acceptance_alpha, self._order_dev, self._lcurve_dev)
        glob.advance(hrows, D)
        return hrows, (float(step_us.max()) * 1e-6 if self.latency is None else None)

    def _emit_trace(self, s, i, out, tmpl, a) -> None:
        tr = out.trace
        alive = tr["alive"][i].astype(bool)
        surv = np.flatnonzero(alive)
        rows = tr["node_row"][i][surv]
        self.trace(self._iteration, {
            "tokens": tr["tokens"][i].tolist(), "positions": tr["positions"][i].tolist(),
            "draft_tokens": tr["draft_tokens"][i].tolist(), "root": int(tr["root"][i]),
            "survivors": surv.tolist(), "argmax": [int(tr["row_argmax"][r]) for r in rows],
            "accepted": [int(v) for v in out.acc_surv[i, :a]], "bonus": int(out.committed[i, a]),
        })

    # ------------------------------------------------------------- plan
    def _plan(self, batch: int, mean_seqlen: float):
        """Static paths, probe queue, or replan (engine.py:307-338)."""
        cfg = self.config
        if not cfg.uses_dynamic:
            return self.static_paths, False
        if self._planned_batch is not None and abs(batch - self._planned_batch) >= cfg.scheduler.resize_batch_delta:
            self.cost.reset()
            self._probe_queue = deque(self.size_candidates * cfg.probe_rounds)
        if self._probe_queue:
            size = self._probe_queue.popleft()
            paths, l = self._select([size])[size]
            self._record_plan("probe", size, {size: l}, batch, mean_seqlen)
            self._selection = paths
            return paths, True
        trigger = self._replan_trigger(batch, mean_seqlen)
        if trigger is None:
            return self._selection, False
        try:
            self.cost.fit(self._iteration)
        except InsufficientDataError:
            pass
        curves = self._select(self.size_candidates)
        l_curve = {s: l for s, (_, l) in curves.items()}
        size = choose_size(l_curve, self.cost, cfg.include_bonus_in_speed)
        self._record_plan(trigger, size, l_curve, batch, mean_seqlen)
        self._selection = curves[size][0]
        return self._selection, True

    def _replan_trigger(self, batch: int, mean_seqlen: float):
        if self._selection is None:
            return "initial"
        sch = self.config.scheduler
        snap = RuntimeSnapshot(batch, mean_seqlen, self._iteration - self._planned_iteration,
                               self._planned_batch if self._planned_batch is not None else batch, self._planned_seqlen)
        if not should_replan(snap, sch):
            return None
        if abs(snap.batch - snap.planned_batch) >= sch.resize_batch_delta:
            return "batch"
        if abs(snap.mean_seqlen - snap.planned_seqlen) >= sch.resize_seqlen_delta:
            return "seqlen"
        return "period"

    def _record_plan(self, trigger, size, l_curve, batch, seqlen) -> None:
        bonus = 1.0 if self.config.include_bonus_in_speed else 0.0
        v_curve = {}
        for s, l in l_curve.items():
            try:
                t = self.cost.estimate(s)
                v_curve[s] = (l + bonus) / t if t > 0 else None
            except InsufficientDataError:
                v_curve[s] = None
        self.plan_events.append(PlanEvent(self._iteration, trigger, size, dict(l_curve), v_curve))
        self._planned_batch, self._planned_seqlen, self._planned_iteration = batch, seqlen, self._iteration

    # ------------------------------------------------------------- helpers
    def _absorb(self, s: _Seq, newly, max_tokens: int) -> int:
        """EOS / max-token clipping of the transcript (engine.py:383-394)."""
        kept = 0
        for tok in newly:
            s.generated.append(int(tok))
            kept += 1
            if (self.config.eos_token is not None and tok == self.config.eos_token) or len(s.generated) >= max_tokens:
                s.finished = True
                break
        return kept

    def _clock(self, wall0: float, rows: float, batch: int, seqlen: float, t_wall: float | None = None) -> float:
        if self.latency is None:
            if t_wall is not None:  # multi-rank: the maximum over ranks, from the step table
                return max(t_wall, 1e-9)
            self.backend.torch.cuda.synchronize(self.backend.device)
            return max(time.perf_counter() - wall0, 1e-9)
        return self.latency.iteration_time(rows, batch=batch, seqlen=seqlen)

    def _summarize(self, metrics) -> RunSummary:
        total_tokens = sum(m.tokens_committed for m in metrics)
        total_time = sum(m.iteration_time for m in metrics)
        tree = [m for m in metrics if m.tree_size > 0]
        mean = (lambda f: float(np.mean([f(m) for m in tree]))) if tree else (lambda f: 0.0)
        return RunSummary(self.config.mode, len(metrics), total_tokens, total_time,
                          total_tokens / total_time if total_time > 0 else 0.0,
                          mean(lambda m: m.mean_accepted), mean(lambda m: m.prune_rate), mean(lambda m: m.tree_size))

    # ------------------------------------------------------------- multi-GPU plumbing
    def _rank_world(self):
        if self.group is None:
            return 0, 1
        import torch.distributed as dist

        return dist.get_rank(self.group), dist.get_world_size(self.group)

def _warm_host_math() -> None:
    """The first weighted least-squares fit initialises numpy's BLAS (tens of
    ms); do it once up front instead of inside the first replanned step."""
    cm = CostModel([1, 2], alpha=1.0, staleness_decay=0.0)
    cm.observe(1, 1.0, now=0)
    cm.observe(2, 2.0, now=0)
    cm.fit(now=1)


def _shard(n: int, rank: int, world: int) -> list:
    """Contiguous index range of batch entries owned by `rank`."""
    lo = (n * rank) // world
    hi = (n * (rank + 1)) // world
    return list(range(lo, hi))


class _Global:
    """Every rank's view of the whole batch chunk in global sequence order
    (committed lengths, active flags, transcripts), advanced from the step
    tables alone."""

    def __init__(self, group, world: int) -> None:
        self.length = [len(p) for p in group]
        self.active = [True] * len(group)
        self.transcripts = [[] for _ in group]
        self.cap = max(1, max(len(_shard(len(group), r, world)) for r in range(world)))

    def any_active(self) -> bool:
        return any(self.active)

    def batch_stats(self):
        lens = [L for L, a in zip(self.length, self.active) if a]
        return len(lens), float(np.mean(lens))

    def advance(self, rows: np.ndarray, D: int) -> None:
        ids = [i for i, a in enumerate(self.active) if a]
        if len(ids) != rows.shape[0]:
            raise RuntimeError(f"step table holds {rows.shape[0]} sequences, {len(ids)} are active")
        for i, r in zip(ids, rows):
            acc = int(r[COL_ACC])
            self.length[i] += acc + 1  # the backend commits the whole chain + bonus (backends.py:337-348)
            self.transcripts[i].extend(int(t) for t in r[COL_RANKS + D: COL_RANKS + D + acc + 1][: int(r[COL_KEPT])])
            self.active[i] = not bool(r[COL_FIN])
