"""Tree templates: the per-step tree SHAPE shared by every sequence.

The reference materialises one TokenTree per sequence per step
(token_tree.py:125-170) and caches the ancestor mask per parents tuple
(engine.py:375-381).  Only the tokens differ between sequences; the shape
(canonical node order, parents, depths, ranks, mask) is a function of the
selected rank paths alone.  `TreeTemplate` computes that shape once per plan
and ships it to the device, where K1 (`propd_tree_embed`) gathers each
sequence's tokens from its draft grid.

Canonical order (token_tree.py:152-169): depth-major; within a depth, by
(parent index, rank).  Ancestor masks are lower-triangular bitsets.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

ROOT = -1


def canonical_order(paths) -> list:
    """Rank paths sorted into the reference's canonical node order."""
    uniq = {tuple(int(r) for r in p) for p in paths}
    kids: dict = {}
    for p in uniq:
        if len(p) == 0:
            raise ValueError("empty rank path")
        if len(p) > 1 and p[:-1] not in uniq:
            raise ValueError(f"path {p}: selection is not ancestor-closed")
        kids.setdefault(p[:-1], []).append(p)
    order: list = []
    level = [()]  # the committed root, outside the tree
    while level:
        # parents are visited in node-index order, children by rank
        level = [c for par in level for c in sorted(kids.get(par, ()), key=lambda q: q[-1])]
        order.extend(level)
    return order


@dataclass(frozen=True)
class TreeTemplate:
    paths: tuple
    parent: np.ndarray
    depth: np.ndarray
    rank: np.ndarray
    mask_bits: np.ndarray  # uint64 [n, W]
    parent_slot: np.ndarray  # index among nodes with children, else -1
    parent_nodes: np.ndarray  # node index of each parent slot
    _dev: dict = field(default_factory=dict, compare=False, repr=False)

    @staticmethod
    def from_paths(paths, depth_count: int | None = None, k_max: int | None = None) -> "TreeTemplate":
        order = canonical_order(paths)
        if not order:
            raise ValueError("a tree needs at least one node")
        for p in order:
            if depth_count is not None and len(p) > depth_count:
                raise ValueError(f"path {p}: depth {len(p)} exceeds {depth_count} heads")
            if k_max is not None and any(not 1 <= r <= k_max for r in p):
                raise ValueError(f"path {p}: ranks must lie in 1..{k_max}")
        index = {p: i for i, p in enumerate(order)}
        n = len(order)
        parent = np.array([index[p[:-1]] if len(p) > 1 else ROOT for p in order], dtype=np.int32)
        depth = np.array([len(p) for p in order], dtype=np.int32)
        rank = np.array([p[-1] for p in order], dtype=np.int32)
        W = (n + 63) // 64
        bits = np.zeros((n, W), dtype=np.uint64)
        for i in range(n):
            if parent[i] >= 0:
                bits[i] = bits[parent[i]]
            bits[i, i // 64] |= np.uint64(1) << np.uint64(i % 64)
        has_child = np.zeros(n, dtype=bool)
        has_child[parent[parent >= 0]] = True
        parent_nodes = np.flatnonzero(has_child).astype(np.int32)
        slot = np.full(n, -1, dtype=np.int32)
        slot[parent_nodes] = np.arange(parent_nodes.size, dtype=np.int32)
        return TreeTemplate(tuple(order), parent, depth, rank, bits, slot, parent_nodes)

    def __len__(self) -> int:
        return len(self.paths)

    @property
    def words(self) -> int:
        return self.mask_bits.shape[1]

    @property
    def max_depth(self) -> int:
        return int(self.depth.max())

    def mask(self) -> np.ndarray:
        """Dense boolean ancestor mask (token_tree.py:173-185 semantics)."""
        n = len(self)
        j = np.arange(n)
        words = self.mask_bits[:, j // 64]
        return ((words >> (j % 64).astype(np.uint64)) & np.uint64(1)).astype(bool)

    def device(self, dev):
        """Device copies (int32 / uint64 tensors), cached per device."""
        import torch

        key = str(dev)
        if key not in self._dev:
            t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
            self._dev[key] = {
                "parent": t(self.parent), "depth": t(self.depth), "rank": t(self.rank),
                "mask": t(self.mask_bits.view(np.int64)), "parent_slot": t(self.parent_slot),
                "parent_nodes": t(self.parent_nodes),
            }
        return self._dev[key]


def mask_to_bits(mask: np.ndarray) -> np.ndarray:
    """Pack an arbitrary boolean [n, n] visibility mask into uint64 bitsets."""
    m = np.asarray(mask, dtype=bool)
    n = m.shape[0]
    W = max(1, (n + 63) // 64)
    padded = np.zeros((n, W * 64), dtype=bool)
    padded[:, :n] = m
    weights = (np.uint64(1) << np.arange(64, dtype=np.uint64))
    return (padded.reshape(n, W, 64).astype(np.uint64) * weights).sum(axis=2, dtype=np.uint64)
