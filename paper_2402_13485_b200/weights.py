"""Model weights: the reference's seeded draw order on the host, or a
same-distribution random init generated directly on the device for large
shapes (7B/33B) where host generation would take minutes.

Reference init (backends.py:165-184): default_rng(seed); emb (V,H), pos
(P,H), then per layer wq, wk, wv, wo (H,H), w1 (H,4H) ~ N(0, 1/sqrt(H)),
w2 (4H,H) ~ N(0, 0.5/sqrt(H)); then w_lm, w_early (H,V), w_draft (D,H,V).
"""

from __future__ import annotations

import numpy as np


def seeded_weights(cfg) -> dict:
    """Host fp64 weights, bit-identical to the reference TinyTransformer(cfg)."""
    g = np.random.default_rng(cfg.seed)
    H, V = cfg.hidden, cfg.vocab
    s = 1.0 / np.sqrt(H)
    out = {"emb": g.normal(0.0, s, size=(V, H)), "pos": g.normal(0.0, s, size=(cfg.max_positions, H))}
    blocks = []
    for _ in range(cfg.layers):
        blk = {name: g.normal(0.0, s, size=(H, H)) for name in ("wq", "wk", "wv", "wo")}
        blk["w1"] = g.normal(0.0, s, size=(H, 4 * H))
        blk["w2"] = g.normal(0.0, 0.5 / np.sqrt(H), size=(4 * H, H))
        blocks.append(blk)
    out["blocks"] = blocks
    out["w_lm"] = g.normal(0.0, s, size=(H, V))
    out["w_early"] = g.normal(0.0, s, size=(H, V))
    out["w_draft"] = g.normal(0.0, s, size=(cfg.draft_heads, H, V))
    return out


def _guard_row(pos):
    """Position table + one zero row at index max_positions: the bonus row of a
    step whose commit would overflow max_positions reads it (in bounds) before
    the host raises the reference's "sequence exceeds max_positions"."""
    import torch

    return torch.cat([pos, torch.zeros(1, pos.shape[1], device=pos.device, dtype=pos.dtype)])


class DeviceWeights:
    """Device-resident weights in the GEMM layout of the B200 path:
    wqkv[l] = [wq | wk | wv] (H, 3H), wo (H, H), w1 (H, 4H), w2 (4H, H),
    w_lm / w_early (H, V), w_draft (H, D*V) with head d in columns [d*V, (d+1)*V)."""

    def __init__(self, cfg, dtype, device, host: dict | None = None, seed: int | None = None) -> None:
        import torch

        self.cfg = cfg
        H, V, D = cfg.hidden, cfg.vocab, cfg.draft_heads
        if host is not None:
            t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device=device, dtype=dtype)
            self.emb, self.pos = t(host["emb"]), _guard_row(t(host["pos"]))
            self.wqkv = [t(np.concatenate([b["wq"], b["wk"], b["wv"]], axis=1)) for b in host["blocks"]]
            self.wo = [t(b["wo"]) for b in host["blocks"]]
            self.w1 = [t(b["w1"]) for b in host["blocks"]]
            self.w2 = [t(b["w2"]) for b in host["blocks"]]
            self.w_lm, self.w_early = t(host["w_lm"]), t(host["w_early"])
            self.w_draft = t(np.concatenate(list(host["w_draft"]), axis=1))
        else:
            g = torch.Generator(device=device)
            g.manual_seed(cfg.seed if seed is None else seed)
            s = 1.0 / float(np.sqrt(H))

            def rnd(rows, cols, std=s):
                w = torch.empty(rows, cols, device=device, dtype=torch.float32)
                w.normal_(0.0, std, generator=g)
                return w.to(dtype)

            self.emb, self.pos = rnd(V, H), _guard_row(rnd(cfg.max_positions, H))
            self.wqkv = [rnd(H, 3 * H) for _ in range(cfg.layers)]
            self.wo = [rnd(H, H) for _ in range(cfg.layers)]
            self.w1 = [rnd(H, 4 * H) for _ in range(cfg.layers)]
            self.w2 = [rnd(4 * H, H, 0.5 * s) for _ in range(cfg.layers)]
            self.w_lm, self.w_early = rnd(H, V), rnd(H, V)
            self.w_draft = rnd(H, D * V)

    def streamed_bytes_per_step(self, prune: bool = True) -> int:
        """Weight bytes one tree step streams from HBM: the layer stack twice
        (tree pass + bonus pass), the LM head twice, the early head once when
        pruning, the draft heads once (the embedding and position tables are
        gathered row by row, not streamed)."""
        el = self.w_lm.element_size()
        layers = self.layer_bytes() * self.cfg.layers
        heads = 2 * self.w_lm.numel() * el + self.w_draft.numel() * el + (self.w_early.numel() * el if prune else 0)
        return 2 * layers + heads

    def nbytes(self) -> int:
        ts = [self.emb, self.pos, self.w_lm, self.w_early, self.w_draft, *self.wqkv, *self.wo, *self.w1, *self.w2]
        return sum(t.numel() * t.element_size() for t in ts)

    def layer_bytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in (self.wqkv[0], self.wo[0], self.w1[0], self.w2[0]))
