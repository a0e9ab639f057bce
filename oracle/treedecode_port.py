"""TEST INFRASTRUCTURE ONLY: float64 numpy restatement of the reference
ProPD decode path (reference package `treedecode`).

Citations `file.py:N` are relative to /root/reference/pkg/src/treedecode/.
This module is the checker for the CUDA path and the CPU baseline timed by
bench.py; the product never imports it.  It is pinned against outputs of the
reference itself (tests/golden/, produced by oracle/make_golden.py).
"""

from __future__ import annotations

import math
import time
from collections import deque
from dataclasses import dataclass, field
from typing import Callable, Iterable, Sequence

import numpy as np

ROOT = -1


# ---------------------------------------------------------------------------
# Model: seeded pre-LN transformer (backends.py:116-348)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class TinyCfg:
    """Mirror of TinyTransformerConfig (backends.py:116-132)."""

    layers: int = 4
    hidden: int = 64
    heads: int = 4
    vocab: int = 256
    draft_heads: int = 4
    max_positions: int = 512
    seed: int = 0


def init_weights(cfg: TinyCfg) -> dict:
    """Seeded weights in the reference draw order (backends.py:165-184)."""
    g = np.random.default_rng(cfg.seed)
    h, v = cfg.hidden, cfg.vocab
    sd = 1.0 / np.sqrt(h)
    w = {"emb": g.normal(0.0, sd, size=(v, h)), "pos": g.normal(0.0, sd, size=(cfg.max_positions, h))}
    layers = []
    for _ in range(cfg.layers):
        blk = {}
        for name in ("wq", "wk", "wv", "wo"):
            blk[name] = g.normal(0.0, sd, size=(h, h))
        blk["w1"] = g.normal(0.0, sd, size=(h, 4 * h))
        blk["w2"] = g.normal(0.0, 0.5 / np.sqrt(h), size=(4 * h, h))
        layers.append(blk)
    w["blocks"] = layers
    w["w_lm"] = g.normal(0.0, sd, size=(h, v))
    w["w_early"] = g.normal(0.0, sd, size=(h, v))
    w["w_draft"] = g.normal(0.0, sd, size=(cfg.draft_heads, h, v))
    return w


def layer_norm(x):
    """No-affine LN, population variance, eps 1e-5 (backends.py:135-138)."""
    mu = x.mean(axis=-1, keepdims=True)
    var = x.var(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + 1e-5)


def gelu_tanh(x):
    """tanh-approximate GELU (backends.py:141-142)."""
    return 0.5 * x * (1.0 + np.tanh(np.sqrt(2.0 / np.pi) * (x + 0.044715 * x**3)))


@dataclass
class SeqState:
    """Per-sequence decode state (backends.py:31-40, 145-150)."""

    committed: list = field(default_factory=list)
    last_tree: tuple | None = None
    kc: list = field(default_factory=list)
    vc: list = field(default_factory=list)
    last_hidden: np.ndarray | None = None
    last_logits: np.ndarray | None = None

    @property
    def length(self) -> int:
        return len(self.committed)


@dataclass(frozen=True)
class TreeFwd:
    """(backends.py:43-50)"""

    survivors: tuple
    argmax: np.ndarray
    logits: np.ndarray | None


def check_chain(mask: np.ndarray, accepted: Sequence[int]) -> None:
    """Accepted path must be a contiguous root chain (backends.py:98-108)."""
    seen: set = set()
    for idx in accepted:
        if idx < 0 or idx >= mask.shape[0]:
            raise ValueError(f"accepted index {idx} outside the verified tree")
        if set(np.flatnonzero(mask[idx]).tolist()) != seen | {idx}:
            raise ValueError("accepted path is not a contiguous root chain")
        seen.add(idx)


class TinyModel:
    """fp64 restatement of TinyTransformer (backends.py:153-348)."""

    def __init__(self, cfg: TinyCfg = TinyCfg(), weights: dict | None = None) -> None:
        self.cfg = cfg
        self.w = weights if weights is not None else init_weights(cfg)

    vocab_size = property(lambda self: self.cfg.vocab)
    num_layers = property(lambda self: self.cfg.layers)
    draft_head_count = property(lambda self: self.cfg.draft_heads)

    def block(self, x, li, kc, vc, vis):
        """One pre-LN block over new rows vs cache + masked new rows (backends.py:202-237)."""
        p = self.w["blocks"][li]
        a = self.cfg.heads
        dh = self.cfg.hidden // a
        n = x.shape[0]
        h = layer_norm(x)
        q, k_new, v_new = h @ p["wq"], h @ p["wk"], h @ p["wv"]
        keys = np.concatenate([kc, k_new], axis=0)
        vals = np.concatenate([vc, v_new], axis=0)
        m = keys.shape[0]
        s = np.einsum("nad,mad->nam", q.reshape(n, a, dh), keys.reshape(m, a, dh)) / np.sqrt(dh)
        visible = np.concatenate([np.ones((n, m - n), dtype=bool), vis], axis=1)
        s = np.where(visible[:, None, :], s, -np.inf)
        s -= s.max(axis=-1, keepdims=True)
        e = np.exp(s)
        pr = e / e.sum(axis=-1, keepdims=True)
        ctx = np.einsum("nam,mad->nad", pr, vals.reshape(m, a, dh)).reshape(n, self.cfg.hidden)
        x = x + ctx @ p["wo"]
        x = x + gelu_tanh(layer_norm(x) @ p["w1"]) @ p["w2"]
        return x, k_new, v_new

    def extend(self, st: SeqState, tokens) -> None:
        """Causal forward of new committed rows, cache append (backends.py:239-259)."""
        toks = np.asarray(tokens, dtype=np.int64)
        if toks.size == 0:
            raise ValueError("cannot extend with zero tokens")
        if np.any((toks < 0) | (toks >= self.cfg.vocab)):
            raise ValueError("token id outside the vocabulary")
        t0, n = st.length, toks.size
        if t0 + n > self.cfg.max_positions:
            raise ValueError("sequence exceeds max_positions")
        x = self.w["emb"][toks] + self.w["pos"][t0 : t0 + n]
        causal = np.tril(np.ones((n, n), dtype=bool))
        for li in range(self.cfg.layers):
            x, kn, vn = self.block(x, li, st.kc[li], st.vc[li], causal)
            st.kc[li] = np.concatenate([st.kc[li], kn], axis=0)
            st.vc[li] = np.concatenate([st.vc[li], vn], axis=0)
        xf = layer_norm(x)
        logits = xf @ self.w["w_lm"]
        st.committed.extend(int(t) for t in toks)
        st.last_hidden = xf[-1]
        st.last_logits = logits[-1]

    def prefill(self, prompt) -> SeqState:
        """(backends.py:263-272)"""
        if len(prompt) == 0:
            raise ValueError("prompt must be non-empty")
        h = self.cfg.hidden
        st = SeqState(kc=[np.zeros((0, h)) for _ in range(self.cfg.layers)],
                      vc=[np.zeros((0, h)) for _ in range(self.cfg.layers)])
        self.extend(st, prompt)
        return st

    def draft(self, st: SeqState, k: int):
        """D draft heads on last_hidden, stable top-k (backends.py:274-285)."""
        if not 1 <= k <= self.cfg.vocab:
            raise ValueError("k outside 1..vocab")
        toks = np.empty((self.cfg.draft_heads, k), dtype=np.int64)
        scores = np.empty((self.cfg.draft_heads, k))
        for d in range(self.cfg.draft_heads):
            lg = st.last_hidden @ self.w["w_draft"][d]
            order = np.argsort(-lg, kind="stable")[:k]
            toks[d], scores[d] = order, lg[order]
        return Preds(toks, scores)

    def next_argmax(self, st: SeqState) -> int:
        """(backends.py:287-288)"""
        return int(np.argmax(st.last_logits))

    def forward_tree(self, st, tokens, positions, mask, *, prune_layer=None, early_topk=0,
                     prune_callback=None) -> TreeFwd:
        """Masked tree pass with optional mid-stack prune (backends.py:290-335)."""
        toks = np.asarray(tokens, dtype=np.int64)
        pos = np.asarray(positions, dtype=np.int64)
        n = toks.size
        if mask.shape != (n, n) or pos.shape != (n,):
            raise ValueError("tokens, positions, and mask sizes disagree")
        if np.any((toks < 0) | (toks >= self.cfg.vocab)):
            raise ValueError("token id outside the vocabulary")
        if np.any(pos < st.length) or np.any(pos >= self.cfg.max_positions):
            raise ValueError("tree positions must follow the committed context")
        if prune_callback is not None:
            if prune_layer is None or not 1 <= prune_layer < self.cfg.layers:
                raise ValueError("prune layer must lie strictly inside the stack")
            if early_topk < 1:
                raise ValueError("early_topk must be positive when pruning")
        x = self.w["emb"][toks] + self.w["pos"][pos]
        vis = mask.astype(bool)
        keep = np.arange(n)
        for li in range(self.cfg.layers):
            x, _, _ = self.block(x, li, st.kc[li], st.vc[li], vis)
            if prune_callback is not None and prune_layer == li + 1:
                early = x @ self.w["w_early"]
                kk = min(early_topk, self.cfg.vocab)
                if getattr(prune_callback, "wants_logits", False):  # probability-based pruning
                    surv = [int(s) for s in prune_callback(early)]
                else:
                    order = np.argsort(-early, axis=1, kind="stable")[:, :kk]
                    surv = [int(s) for s in prune_callback([r.tolist() for r in order])]
                vis = subsample_mask(vis, surv)
                x, keep = x[surv], keep[surv]
        logits = layer_norm(x) @ self.w["w_lm"]
        st.last_tree = (toks[keep].copy(), vis.copy())
        return TreeFwd(tuple(int(i) for i in keep), np.argmax(logits, axis=1).astype(np.int64), logits)

    def commit(self, st: SeqState, accepted, bonus) -> None:
        """Validate the chain, recompute accepted + bonus rows (backends.py:337-348)."""
        acc = [int(a) for a in accepted]
        if acc:
            if st.last_tree is None:
                raise ValueError("commit with accepted nodes needs a preceding tree forward")
            ttoks, tmask = st.last_tree
            check_chain(tmask, acc)
            new = [int(ttoks[i]) for i in acc] + [int(bonus)]
        else:
            new = [int(bonus)]
        self.extend(st, new)
        st.last_tree = None


class Clock:
    """Simulated affine iteration clock (backends.py:568-603)."""

    def __init__(self, c0_base=1.0, c0_batch=0.0, c0_seqlen=0.0, c1_base=0.05, c1_batch=0.0,
                 noise=0.0, seed=0):
        if noise < 0.0:
            raise ValueError("noise amplitude must be non-negative")
        self.c = (float(c0_base), float(c0_batch), float(c0_seqlen), float(c1_base), float(c1_batch))
        self.noise = float(noise)
        self.rng = np.random.default_rng(seed)

    def iteration_time(self, rows, batch=1, seqlen=0.0) -> float:
        c0b, c0B, c0s, c1b, c1B = self.c
        t = (c0b + c0B * batch + c0s * seqlen) + (c1b + c1B * batch) * float(rows)
        if self.noise > 0.0:
            t += float(self.rng.uniform(-self.noise, self.noise))
        if t <= 0.0:
            raise ValueError("latency coefficients produced a non-positive time")
        return float(t)


# ---------------------------------------------------------------------------
# Trees (token_tree.py:32-226)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class Node:
    token: int
    parent: int
    depth: int
    rank: int
    weight: float = 1.0


@dataclass(frozen=True)
class Tree:
    """Canonically ordered token tree (token_tree.py:48-122)."""

    nodes: tuple
    root_token: int

    def __len__(self):
        return len(self.nodes)

    tokens = property(lambda self: np.array([n.token for n in self.nodes], dtype=np.int64))
    parents = property(lambda self: np.array([n.parent for n in self.nodes], dtype=np.int64))
    depths = property(lambda self: np.array([n.depth for n in self.nodes], dtype=np.int64))

    def children(self):
        kids = [[] for _ in self.nodes]
        for i, nd in enumerate(self.nodes):
            if nd.parent != ROOT:
                kids[nd.parent].append(i)
        return kids

    def roots(self):
        return [i for i, nd in enumerate(self.nodes) if nd.parent == ROOT]

    def ancestors(self, i):
        out = []
        p = self.nodes[i].parent
        while p != ROOT:
            out.append(p)
            p = self.nodes[p].parent
        return out[::-1]


def build_tree(preds, selected: Iterable, *, root_token: int, weights=None) -> Tree:
    """Depth-major, siblings by (parent index, rank) (token_tree.py:125-170)."""
    paths = {tuple(int(r) for r in p) for p in selected}
    for p in paths:
        if not p:
            raise ValueError("empty rank path")
        if len(p) > preds.depth_count:
            raise ValueError(f"path {p}: depth {len(p)} exceeds {preds.depth_count} heads")
        if any(not 1 <= r <= preds.k_max for r in p):
            raise ValueError(f"path {p}: ranks must lie in 1..{preds.k_max}")
        if len(p) > 1 and p[:-1] not in paths:
            raise ValueError(f"path {p}: selection is not ancestor-closed")
    where: dict = {}
    nodes: list = []
    top = max((len(p) for p in paths), default=0)
    for d in range(1, top + 1):
        layer = sorted((p for p in paths if len(p) == d),
                       key=lambda p: (where[p[:-1]] if d > 1 else ROOT, p[-1]))
        for p in layer:
            par = where[p[:-1]] if d > 1 else ROOT
            wt = 1.0 if weights is None else float(weights[p])
            nodes.append(Node(int(preds.token(d, p[-1])), par, d, p[-1], wt))
            where[p] = len(nodes) - 1
    return Tree(tuple(nodes), int(root_token))


def make_mask(tree: Tree) -> np.ndarray:
    """mask[i, j] iff j is i or an ancestor of i (token_tree.py:173-185)."""
    n = len(tree)
    m = np.zeros((n, n), dtype=bool)
    for i, nd in enumerate(tree.nodes):
        if nd.parent != ROOT:
            m[i, :i] = m[nd.parent, :i]
        m[i, i] = True
    return m


def subsample_mask(mask: np.ndarray, survivors) -> np.ndarray:
    """Row/column gather onto an ancestor-closed survivor set (token_tree.py:188-207)."""
    n = mask.shape[0]
    s = np.asarray(survivors, dtype=np.int64)
    if s.ndim != 1:
        raise ValueError("survivors must be a flat index list")
    if s.size and (s[0] < 0 or s[-1] >= n):
        raise ValueError("survivor index out of range")
    if np.any(np.diff(s) <= 0):
        raise ValueError("survivors must be strictly increasing")
    kept = np.zeros(n, dtype=bool)
    kept[s] = True
    for i in s:
        if not np.all(kept[mask[i]]):
            raise ValueError(f"survivor {i}: an ancestor was dropped (set is not ancestor-closed)")
    return mask[np.ix_(s, s)].copy()


def restrict(tree: Tree, survivors) -> Tree:
    """Induced subtree on survivors (token_tree.py:210-226)."""
    s = [int(i) for i in survivors]
    if any(b <= a for a, b in zip(s, s[1:])):
        raise ValueError("survivors must be strictly increasing")
    remap = {old: new for new, old in enumerate(s)}
    out = []
    for old in s:
        nd = tree.nodes[old]
        if nd.parent == ROOT:
            par = ROOT
        elif nd.parent in remap:
            par = remap[nd.parent]
        else:
            raise ValueError(f"survivor {old}: parent {nd.parent} was dropped")
        out.append(Node(nd.token, par, nd.depth, nd.rank, nd.weight))
    return Tree(tuple(out), tree.root_token)


def complete_tree_paths(depth_count: int, k_max: int) -> list:
    """Every rank path of the k^D universe, depth-major (token_tree.py:251-258)."""
    out, level = [], [()]
    for _ in range(depth_count):
        level = [p + (r,) for p in level for r in range(1, k_max + 1)]
        out.extend(level)
    return out


def format_mask(mask: np.ndarray) -> str:
    """(token_tree.py:286-291)"""
    return "\n".join([str(mask.shape[0])] + ["".join(str(int(v)) for v in row) for row in mask]) + "\n"


# ---------------------------------------------------------------------------
# Pruning and verification (pruning.py:40-73, verification.py:30-53)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class PruneCfg:
    layer: int = 4
    topk: int = 50
    threshold: float | None = None  # probability-based pruning (probability_prune) when set


def prune(tree: Tree, early_lists, cfg: PruneCfg):
    """Top-down survival: depth-1 exempt, else parent alive and token in the
    parent's early list (pruning.py:40-66).  Returns (survivors, rate)."""
    n = len(tree)
    if len(early_lists) != n:
        raise ValueError("early_topk must have one list per tree node")
    sets = []
    for i, lst in enumerate(early_lists):
        st = {int(t) for t in lst}
        if len(st) != len(lst):
            raise ValueError(f"node {i}: early top-K list has duplicates")
        if len(lst) > cfg.topk:
            raise ValueError(f"node {i}: early list longer than top-K = {cfg.topk}")
        sets.append(st)
    alive = np.zeros(n, dtype=bool)
    for i, nd in enumerate(tree.nodes):
        alive[i] = True if nd.parent == ROOT else bool(alive[nd.parent] and nd.token in sets[nd.parent])
    surv = tuple(int(i) for i in np.flatnonzero(alive))
    return surv, (0.0 if n == 0 else 1.0 - len(surv) / n)


def row_lse_entropy(logits, temperature: float = 1.0):
    """Per row of z = logits / T: log-sum-exp and entropy H = lse - sum(p z) (fp64)."""
    z = np.asarray(logits, dtype=np.float64) / float(temperature)
    m = z.max(axis=1, keepdims=True)
    e = np.exp(z - m)
    s = e.sum(axis=1, keepdims=True)
    lse = (m + np.log(s))[:, 0]
    H = lse - (e * z).sum(axis=1) / s[:, 0]
    return lse, H


def probability_prune(tree: Tree, early_logits, threshold: float):
    """Probability-based early pruning (the reference ships
    only top-K and disables this entry point, pruning.py:76-82 -- parity
    unpinned, this restatement is the definition the B200 kernel follows): a
    node survives iff it has depth 1, or its parent survives and the marginal
    path probability prod p_early(token | parent row) >= threshold.  Terms are
    summed top-down in log space in fp64.  Returns (survivors, rate)."""
    n = len(tree)
    early = np.asarray(early_logits, dtype=np.float64)
    lse, _ = row_lse_entropy(early)
    log_tau = math.log(threshold)
    logp = np.zeros(n)
    alive = np.zeros(n, dtype=bool)
    for i, nd in enumerate(tree.nodes):
        if nd.parent == ROOT:
            alive[i] = True
        else:
            logp[i] = logp[nd.parent] + (early[nd.parent, nd.token] - lse[nd.parent])
            alive[i] = bool(alive[nd.parent] and logp[i] >= log_tau)
    surv = tuple(int(i) for i in np.flatnonzero(alive))
    return surv, (0.0 if n == 0 else 1.0 - len(surv) / n)


def typical_verify(tree: Tree, node_logits, root_logits, epsilon: float, alpha: float, temperature: float = 1.0):
    """Typical acceptance (Medusa-style; named by the north star, absent from
    the reference -- parity unpinned, this restatement is the definition the
    B200 kernel follows): with p = softmax(logits / T) of the accepting row,
    candidate token x is typical iff log p(x) > min(log eps, log alpha - H(p)).
    A node is accepted iff it is typical under its parent's row (depth 1:
    under the root row = the last committed token's logits) and its parent is
    accepted.  The path to the deepest accepted node (ties: lowest index) is
    committed; the bonus is the argmax of that node's row (root row if none).
    Returns (accepted, bonus)."""
    n = len(tree)
    rows = np.asarray(node_logits, dtype=np.float64)
    root = np.asarray(root_logits, dtype=np.float64)[None, :]
    lse, H = row_lse_entropy(rows, temperature) if n else (np.zeros(0), np.zeros(0))
    rlse, rH = row_lse_entropy(root, temperature)
    le = math.log(epsilon)
    la = math.log(alpha)

    def typical(z_row, lse_r, H_r, tok):
        return (z_row[tok] / temperature - lse_r) > min(le, la - H_r)

    acc = np.zeros(n, dtype=bool)
    for i, nd in enumerate(tree.nodes):
        if nd.parent == ROOT:
            acc[i] = typical(root[0], rlse[0], rH[0], nd.token)
        else:
            acc[i] = bool(acc[nd.parent] and typical(rows[nd.parent], lse[nd.parent], H[nd.parent], nd.token))
    depths = tree.depths
    best, best_d = -1, 0
    for i in range(n):
        if acc[i] and int(depths[i]) > best_d:
            best, best_d = i, int(depths[i])
    if best < 0:
        return (), int(np.argmax(root[0]))
    chain = []
    j = best
    while j != ROOT:
        chain.append(j)
        j = tree.nodes[j].parent
    return tuple(reversed(chain)), int(np.argmax(rows[best]))


def verify(tree: Tree, node_argmax, root_argmax: int):
    """Greedy root-chain walk (verification.py:30-53).  Returns (accepted, bonus)."""
    if len(node_argmax) != len(tree):
        raise ValueError("node_argmax must align with the tree's nodes")
    kids = tree.children()
    frontier = tree.roots()
    target = int(root_argmax)
    acc = []
    while True:
        hit = next((i for i in frontier if tree.nodes[i].token == target), None)
        if hit is None:
            return tuple(acc), target
        acc.append(hit)
        target = int(node_argmax[hit])
        frontier = kids[hit]


# ---------------------------------------------------------------------------
# Acceptance model (acceptance.py:20-206)
# ---------------------------------------------------------------------------


class Preds:
    """Per-head top-k grid (acceptance.py:20-57)."""

    def __init__(self, tokens, scores):
        self.tokens = np.asarray(tokens, dtype=np.int64)
        self.scores = np.asarray(scores, dtype=np.float64)
        if self.tokens.ndim != 2 or self.tokens.shape != self.scores.shape:
            raise ValueError("tokens and scores must be matching 2-D arrays")
        for d, row in enumerate(self.tokens, start=1):
            if len(set(row.tolist())) != row.size:
                raise ValueError(f"head {d}: duplicate tokens in the top-k list")
        if np.any(np.diff(self.scores, axis=1) > 0):
            raise ValueError("scores must be non-increasing within each head")

    depth_count = property(lambda self: self.tokens.shape[0])
    k_max = property(lambda self: self.tokens.shape[1])

    def token(self, depth, rank):
        if not (1 <= depth <= self.depth_count and 1 <= rank <= self.k_max):
            raise IndexError(f"no prediction at depth {depth}, rank {rank}")
        return int(self.tokens[depth - 1, rank - 1])

    def rank_of(self, depth, token):
        hits = np.flatnonzero(self.tokens[depth - 1] == token)
        return int(hits[0]) + 1 if hits.size else None


class Stats:
    """Cumulative top-k hit curves per head (acceptance.py:60-145)."""

    def __init__(self, depth_count, k_max, alpha=0.05, prewarm=True):
        if depth_count < 1 or k_max < 1:
            raise ValueError("depth_count and k_max must be positive")
        if alpha is not None and not 0.0 < alpha <= 1.0:
            raise ValueError("alpha must lie in (0, 1] or be None")
        self.alpha = alpha
        self.counts = np.zeros(depth_count, dtype=np.int64)
        if prewarm:
            cap = np.minimum(0.9, 0.5 ** np.arange(1, depth_count + 1))
            self.P = np.outer(cap, np.arange(1, k_max + 1) / k_max)
        else:
            self.P = np.zeros((depth_count, k_max))

    depth_count = property(lambda self: self.P.shape[0])
    k_max = property(lambda self: self.P.shape[1])

    def update(self, realized: dict, preds: Preds) -> None:
        """EMA / running-mean step per known depth (acceptance.py:96-113)."""
        if preds.depth_count != self.depth_count or preds.k_max != self.k_max:
            raise ValueError("predictions shape does not match the tracked grid")
        for depth, tok in realized.items():
            if not 1 <= depth <= self.depth_count:
                raise ValueError(f"depth {depth} outside 1..{self.depth_count}")
            r = preds.rank_of(depth, tok)
            hit = np.zeros(self.k_max)
            if r is not None:
                hit[r - 1:] = 1.0
            self.counts[depth - 1] += 1
            step = self.alpha if self.alpha is not None else 1.0 / self.counts[depth - 1]
            self.P[depth - 1] = (1.0 - step) * self.P[depth - 1] + step * hit

    def marginals(self):
        return np.diff(self.P, axis=1, prepend=0.0)

    def marginal(self, depth, rank):
        lo = self.P[depth - 1, rank - 2] if rank > 1 else 0.0
        return float(self.P[depth - 1, rank - 1] - lo)

    def path_contribution(self, path):
        v = 1.0
        for i, (d, r) in enumerate(path, start=1):
            if d != i:
                raise ValueError("path depths must be consecutive starting at 1")
            v *= self.marginal(d, r)
        return v


def grid_candidates(depth_count, k_max):
    """Spine + side-branch universe (1,...,1,k) (acceptance.py:158-169)."""
    return tuple((1,) * (d - 1) + (r,) for d in range(1, depth_count + 1) for r in range(1, k_max + 1))


def select_best_nodes(stats: Stats, sizes):
    """Greedy top-i by contribution; {size: (paths, l)} (acceptance.py:186-206)."""
    cap = stats.depth_count * stats.k_max
    for s in sizes:
        if not 1 <= s <= cap:
            raise ValueError(f"size {s} outside the 1..{cap} grid capacity")
    m = stats.marginals()
    spine = np.concatenate([[1.0], np.cumprod(m[:, 0])])
    cands = grid_candidates(stats.depth_count, stats.k_max)
    contrib = {p: float(spine[len(p) - 1] * m[len(p) - 1, p[-1] - 1]) for p in cands}
    order = sorted(cands, key=lambda p: (-contrib[p], len(p), p[-1]))
    return {s: (tuple(order[:s]), float(sum(contrib[p] for p in order[:s]))) for s in sizes}


# ---------------------------------------------------------------------------
# Cost model and scheduler (cost_model.py:26-118, scheduler.py:41-77)
# ---------------------------------------------------------------------------


class NoFit(RuntimeError):
    """(cost_model.py:22-23)"""


class Cost:
    def __init__(self, sizes, alpha=0.2, staleness_decay=0.01):
        self.sizes = sorted({int(s) for s in sizes})
        self.alpha, self.decay = alpha, staleness_decay
        self.t: dict = {}
        self.last: dict = {}
        self.beta = None

    def observe(self, size, t, now):
        """(cost_model.py:49-62)"""
        if size not in set(self.sizes):
            raise ValueError(f"size {size} is not a tracked candidate")
        prev = self.t.get(size)
        self.t[size] = float(t) if prev is None else (1.0 - self.alpha) * prev + self.alpha * float(t)
        self.last[size] = int(now)

    def weights(self, now):
        """(cost_model.py:68-75)"""
        w = np.zeros(len(self.sizes))
        for i, s in enumerate(self.sizes):
            if s in self.last:
                w[i] = math.exp(-self.decay * (int(now) - self.last[s]))
        return w

    def fit(self, now):
        """Closed-form weighted least squares (cost_model.py:77-102)."""
        w = self.weights(now)
        on = w > 0.0
        xs = np.array(self.sizes, dtype=np.float64)[on]
        if np.unique(xs).size < 2:
            raise NoFit("need observations at two distinct sizes to fit a line")
        ys = np.array([self.t[s] for s, a in zip(self.sizes, on) if a])
        ww = w[on]
        sw = ww.sum()
        sx, sy = float(ww @ xs), float(ww @ ys)
        sxx, sxy = float(ww @ (xs * xs)), float(ww @ (xs * ys))
        den = sw * sxx - sx * sx
        if den <= 0.0:
            raise NoFit("degenerate design: distinct sizes collapsed")
        slope = (sw * sxy - sx * sy) / den
        self.beta = ((sy - slope * sx) / sw, slope)
        return self.beta

    def estimate(self, size):
        if self.beta is None:
            raise NoFit("no fit has succeeded and no pre-warm line is set")
        return self.beta[0] + self.beta[1] * float(size)

    def reset(self):
        self.t.clear()
        self.last.clear()


def choose_size(l_curve: dict, cost: Cost, include_bonus=False) -> int:
    """Ascending scan, strict improvement (scheduler.py:41-69)."""
    best, best_v = None, None
    for s in sorted(l_curve):
        try:
            t = cost.estimate(s)
        except NoFit:
            break
        if t <= 0.0:
            continue
        v = (l_curve[s] + (1.0 if include_bonus else 0.0)) / t
        if best_v is None or v > best_v:
            best, best_v = s, v
    return min(l_curve) if best is None else best


# ---------------------------------------------------------------------------
# Decode engine (engine.py:31-414)
# ---------------------------------------------------------------------------

MODES = ("autoregressive", "static_tree", "prune_only", "dynamic_only", "propd_full")


@dataclass(frozen=True)
class SchedCfg:
    resize_batch_delta: int = 1
    resize_seqlen_delta: int = 256
    replan_period: int = 16
    size_candidates: tuple = (1, 2, 4, 8, 16, 32, 64)


@dataclass(frozen=True)
class EngineCfg:
    mode: str = "propd_full"
    draft_heads: int = 4
    draft_topk: int = 3
    prune: PruneCfg | None = None
    scheduler: SchedCfg = SchedCfg()
    static_tree: tuple | None = None
    acceptance_alpha: float | None = 0.05
    cost_alpha: float = 0.2
    cost_staleness: float = 0.01
    include_bonus_in_speed: bool = False
    probe_rounds: int = 1
    eos_token: int | None = None
    acceptance: str = "greedy"  # or "typical" (typical_verify)
    typical_epsilon: float = 0.09
    typical_alpha: float = 0.3
    typical_temperature: float = 1.0

    uses_tree = property(lambda self: self.mode != "autoregressive")
    uses_prune = property(lambda self: self.mode in ("prune_only", "propd_full"))
    uses_dynamic = property(lambda self: self.mode in ("dynamic_only", "propd_full"))


METRIC_KEYS = ("iteration", "batch", "mean_seqlen", "tree_size", "mean_survivors", "prune_rate",
               "mean_accepted", "tokens_committed", "iteration_time", "replanned")


class Engine:
    """Restatement of DecodeEngine (engine.py:139-414).  `trace` (optional
    callable) receives a per-sequence record of every tree step."""

    def __init__(self, backend, cfg: EngineCfg, clock: Clock | None = None,
                 trace: Callable | None = None):
        self.b, self.cfg, self.clock, self.trace = backend, cfg, clock, trace
        grid = cfg.draft_heads * cfg.draft_topk
        self.size_candidates = sorted({min(int(s), grid) for s in cfg.scheduler.size_candidates})
        if cfg.mode in ("static_tree", "prune_only"):
            self.static_paths = cfg.static_tree if cfg.static_tree is not None else grid_candidates(
                cfg.draft_heads, cfg.draft_topk)
        else:
            self.static_paths = ()
        sizes = set(self.size_candidates) | ({len(self.static_paths)} if self.static_paths else set())
        self.stats = Stats(cfg.draft_heads, cfg.draft_topk, alpha=cfg.acceptance_alpha)
        self.cost = Cost(sizes, alpha=cfg.cost_alpha, staleness_decay=cfg.cost_staleness)
        self.masks: dict = {}
        self.it = 0
        self.selection = None
        self.planned_batch = None
        self.planned_seqlen = 0.0
        self.planned_it = 0
        self.probes = deque(self.size_candidates * cfg.probe_rounds)
        self.plan_events: list = []

    def run(self, prompts, max_tokens, batch_size=None):
        """Chunked batches; estimator state carries across chunks (engine.py:189-221)."""
        if max_tokens < 1:
            raise ValueError("max_tokens must be positive")
        prompts = [list(map(int, p)) for p in prompts]
        if not prompts or any(len(p) == 0 for p in prompts):
            raise ValueError("prompts must be non-empty")
        chunk = len(prompts) if batch_size is None else max(1, int(batch_size))
        transcripts, metrics = [], []
        for lo in range(0, len(prompts), chunk):
            seqs = [{"state": self.b.prefill(p), "prompt": p, "gen": [], "done": False}
                    for p in prompts[lo: lo + chunk]]
            active = list(seqs)
            while active:
                metrics.append(self.step(active, max_tokens))
                active = [s for s in seqs if not s["done"]]
            transcripts.extend(s["gen"] for s in seqs)
        tot_tok = sum(m["tokens_committed"] for m in metrics)
        tot_t = sum(m["iteration_time"] for m in metrics)
        tree_rows = [m for m in metrics if m["tree_size"] > 0]
        mean = lambda key: float(np.mean([m[key] for m in tree_rows])) if tree_rows else 0.0
        summary = {"mode": self.cfg.mode, "iterations": len(metrics), "total_tokens": tot_tok,
                   "total_time": tot_t, "tokens_per_sec": tot_tok / tot_t if tot_t > 0 else 0.0,
                   "mean_accepted": mean("mean_accepted"), "mean_prune_rate": mean("prune_rate"),
                   "mean_tree_size": mean("tree_size")}
        return {"transcripts": transcripts, "prompts": prompts, "metrics": metrics,
                "plan_events": list(self.plan_events), "summary": summary}

    def _metric(self, *vals):
        return dict(zip(METRIC_KEYS, vals))

    def step(self, active, max_tokens):
        """One iteration (engine.py:225-303)."""
        self.it += 1
        B = len(active)
        seqlen = float(np.mean([s["state"].length for s in active]))
        t_wall = time.perf_counter() if self.clock is None else 0.0
        cfg = self.cfg
        if not cfg.uses_tree:
            n_tok = 0
            for s in active:
                tok = self.b.next_argmax(s["state"])
                self.b.commit(s["state"], [], tok)
                n_tok += self._absorb(s, [tok], max_tokens)
            t = self._time(t_wall, 1.0, B, seqlen)
            return self._metric(self.it, B, seqlen, 0, 0.0, 0.0, 0.0, n_tok, t, False)
        drafts = [self.b.draft(s["state"], cfg.draft_topk) for s in active]
        roots = [self.b.next_argmax(s["state"]) for s in active]
        paths, replanned = self._plan(B, seqlen)
        weights = ({p: self.stats.path_contribution(list(enumerate(p, start=1))) for p in paths}
                   if cfg.uses_dynamic else None)
        n = len(paths)
        surv_tot = acc_tot = n_tok = 0
        rates = []
        for s, pred, root in zip(active, drafts, roots):
            st = s["state"]
            last_tok = s["gen"][-1] if s["gen"] else s["prompt"][-1]
            tree = build_tree(pred, paths, root_token=last_tok, weights=weights)
            key = tuple(int(p) for p in tree.parents)
            if key not in self.masks:
                self.masks[key] = make_mask(tree)
            mask = self.masks[key]
            positions = st.length + tree.depths - 1
            rec = {"tokens": tree.tokens.tolist(), "parents": tree.parents.tolist(),
                   "positions": positions.tolist(), "length": st.length}
            if cfg.uses_prune:
                box = {}

                def on_early(lists, _t=tree, _b=box):
                    _b["lists"] = lists
                    if cfg.prune.threshold is not None:
                        _b["dec"] = probability_prune(_t, lists, cfg.prune.threshold)
                    else:
                        _b["dec"] = prune(_t, lists, cfg.prune)
                    return _b["dec"][0]

                on_early.wants_logits = cfg.prune.threshold is not None

                fwd = self.b.forward_tree(st, tree.tokens, positions, mask, prune_layer=cfg.prune.layer,
                                          early_topk=cfg.prune.topk, prune_callback=on_early)
                surv, rate = box["dec"]
                vtree = restrict(tree, surv)
                subsample_mask(mask, surv)
                rates.append(rate)
                rec["early_lists"] = (box["lists"] if cfg.prune.threshold is None
                                      else np.argsort(-box["lists"], axis=1, kind="stable")[:, :4].tolist())
            else:
                fwd = self.b.forward_tree(st, tree.tokens, positions, mask)
                vtree = tree
            if cfg.acceptance == "typical":
                accepted, bonus = typical_verify(vtree, fwd.logits, st.last_logits, cfg.typical_epsilon,
                                                 cfg.typical_alpha, cfg.typical_temperature)
            else:
                accepted, bonus = verify(vtree, fwd.argmax, root)
            self.b.commit(st, accepted, bonus)
            newly = [vtree.nodes[i].token for i in accepted] + [bonus]
            n_tok += self._absorb(s, newly, max_tokens)
            acc_tot += len(accepted)
            surv_tot += len(fwd.survivors)
            realized = {d: newly[d - 1] for d in range(1, min(len(newly), cfg.draft_heads) + 1)}
            self.stats.update(realized, pred)
            if self.trace is not None:
                rec.update(survivors=list(fwd.survivors), argmax=[int(a) for a in fwd.argmax],
                           accepted=list(accepted), bonus=int(bonus), root=int(root),
                           draft_tokens=pred.tokens.tolist())
                self.trace(self.it, rec)
        surv_mean = surv_tot / B
        if cfg.uses_prune:
            p, L = cfg.prune.layer, self.b.num_layers
            rows = (p * n + (L - p) * surv_mean) / L
        else:
            rows = float(n)
        t = self._time(t_wall, rows, B, seqlen)
        self.cost.observe(n, t, now=self.it)
        return self._metric(self.it, B, seqlen, n, surv_mean,
                            float(np.mean(rates)) if rates else 0.0, acc_tot / B, n_tok, t, replanned)

    def _plan(self, B, seqlen):
        """Static paths, probe queue, or replan (engine.py:307-338)."""
        cfg = self.cfg
        if not cfg.uses_dynamic:
            return self.static_paths, False
        if self.planned_batch is not None and abs(B - self.planned_batch) >= cfg.scheduler.resize_batch_delta:
            self.cost.reset()
            self.probes = deque(self.size_candidates * cfg.probe_rounds)
        if self.probes:
            size = self.probes.popleft()
            paths, l = select_best_nodes(self.stats, [size])[size]
            self._record("probe", size, {size: l}, B, seqlen)
            self.selection = paths
            return paths, True
        trig = self._trigger(B, seqlen)
        if trig is None:
            return self.selection, False
        try:
            self.cost.fit(self.it)
        except NoFit:
            pass
        curves = select_best_nodes(self.stats, self.size_candidates)
        lc = {s: l for s, (_, l) in curves.items()}
        size = choose_size(lc, self.cost, cfg.include_bonus_in_speed)
        self._record(trig, size, lc, B, seqlen)
        self.selection = curves[size][0]
        return self.selection, True

    def _trigger(self, B, seqlen):
        """(engine.py:340-356, scheduler.py:72-77)"""
        if self.selection is None:
            return "initial"
        sch = self.cfg.scheduler
        pb = self.planned_batch if self.planned_batch is not None else B
        db, ds = abs(B - pb), abs(seqlen - self.planned_seqlen)
        if not (db >= sch.resize_batch_delta or ds >= sch.resize_seqlen_delta
                or self.it - self.planned_it >= sch.replan_period):
            return None
        if db >= sch.resize_batch_delta:
            return "batch"
        if ds >= sch.resize_seqlen_delta:
            return "seqlen"
        return "period"

    def _record(self, trig, size, lc, B, seqlen):
        """(engine.py:358-371)"""
        vc = {}
        for s, l in lc.items():
            try:
                t = self.cost.estimate(s)
                vc[s] = (l + (1.0 if self.cfg.include_bonus_in_speed else 0.0)) / t if t > 0 else None
            except NoFit:
                vc[s] = None
        self.plan_events.append({"iteration": self.it, "trigger": trig, "chosen_size": size,
                                 "l_curve": dict(lc), "v_curve": vc})
        self.planned_batch, self.planned_seqlen, self.planned_it = B, seqlen, self.it

    def _absorb(self, s, newly, max_tokens):
        """EOS / max-token clip after the full commit (engine.py:383-394)."""
        kept = 0
        for tok in newly:
            s["gen"].append(int(tok))
            kept += 1
            if self.cfg.eos_token is not None and tok == self.cfg.eos_token:
                s["done"] = True
                break
            if len(s["gen"]) >= max_tokens:
                s["done"] = True
                break
        return kept

    def _time(self, t_wall, rows, B, seqlen):
        if self.clock is None:
            return max(time.perf_counter() - t_wall, 1e-9)
        return self.clock.iteration_time(rows, batch=B, seqlen=seqlen)


def greedy_transcript(backend, prompt, max_tokens, eos=None):
    """One-token-at-a-time greedy stream (tests/oracles.py:65-75)."""
    st = backend.prefill(list(prompt))
    out = []
    while len(out) < max_tokens:
        tok = backend.next_argmax(st)
        backend.commit(st, [], tok)
        out.append(int(tok))
        if eos is not None and tok == eos:
            break
    return out


RUN_TINY = {
    # configs/run_tiny.json (+ config.py:173-207 defaults, latency seed = backend seed + 1)
    "model": TinyCfg(layers=4, hidden=64, heads=4, vocab=256, draft_heads=4, max_positions=512, seed=3),
    "clock": dict(c0_base=3.0, c1_base=0.05, noise=0.02, seed=4),
    "engine": EngineCfg(mode="propd_full", draft_heads=4, draft_topk=3, prune=PruneCfg(layer=2, topk=24),
                        scheduler=SchedCfg(replan_period=16, size_candidates=(1, 2, 4, 6, 8, 10, 12))),
    "workload": dict(num_prompts=8, prompt_len=6, max_tokens=32, batch_size=4, seed=5),
}


def synthetic_prompts(vocab, num_prompts, prompt_len, seed):
    """Uniform random prompts (config.py:350-354)."""
    g = np.random.default_rng(seed)
    return [g.integers(0, vocab, size=prompt_len).tolist() for _ in range(num_prompts)]
