"""TEST INFRASTRUCTURE ONLY: teacher-forced step parity of the batched B200
tree step (bf16 performance mode) against the fp64 oracle.

One call runs `B200Backend.step_tree` over the whole batch (the product path:
graphs, device row counts, tcgen05 attention / weight-streaming projections,
K3 prune, K5 accept + KV compaction, bonus pass) and replays each sequence's
step on the oracle (`oracle.treedecode_port.TinyModel`, the fp64 restatement
of the reference's `DecodeEngine._step` body, engine.py:243-303) with the
device's decisions fed in wherever bf16 rounding could legitimately flip
them:

* the tree is built from the device's draft tokens (backends.py:274-285),
* the mid-stack prune callback (backends.py:320-327) returns the device's
  survivor set, so logits are compared row for row,
* the oracle commits the device's accepted chain + bonus (backends.py:337-348).

Every decision is then compared with the oracle's own where the oracle's
decision margin exceeds twice the error measured on the values behind it
(draft ranks, the early-head membership test, the root and row argmaxes, the
greedy walk, verification.py:30-53); the undecidable fraction is reported.
Only tests/ and __graft_entry__.smoke() import this module.
"""

from __future__ import annotations

import numpy as np

from . import treedecode_port as op


def _top2_gap(rows: np.ndarray) -> np.ndarray:
    t = np.sort(rows, axis=-1)[..., -2:]
    return t[..., 1] - t[..., 0]


class _Replay:
    """prune_callback with wants_logits: records the oracle's early logits and
    returns the device's (ancestor-closed) survivor set."""

    wants_logits = True

    def __init__(self, survivors):
        self.survivors = survivors
        self.early = None

    def __call__(self, early):
        self.early = np.array(early, copy=True)
        return self.survivors


class StepReport:
    def __init__(self) -> None:
        self.n = {"draft": [0, 0], "root": [0, 0], "member": [0, 0], "argmax": [0, 0], "walk": [0, 0]}
        self.err = {"draft": 0.0, "early": 0.0, "logits": 0.0}
        self.scale = {"draft": 0.0, "early": 0.0, "logits": 0.0}
        self.accepted = 0

    def count(self, key, decidable, total):
        self.n[key][0] += int(decidable)
        self.n[key][1] += int(total)

    def frac(self, key):
        d, t = self.n[key]
        return d / t if t else 1.0

    def summary(self) -> dict:
        return {"decidable": {k: f"{d}/{t}" for k, (d, t) in self.n.items()},
                "max_err": dict(self.err), "ref_scale": dict(self.scale), "accepted": self.accepted}


def _note_err(rep, key, dev, ref):
    rep.err[key] = max(rep.err[key], float(np.abs(np.asarray(dev, np.float64) - ref).max()))
    rep.scale[key] = max(rep.scale[key], float(np.abs(ref).max()))


def teacher_forced_step(be, ref: op.TinyModel, states, ref_states, tmpl, k: int, prune=None,
                        rel_tol: float = 5e-2, rep: StepReport | None = None) -> StepReport:
    """One batched device step vs the oracle; raises AssertionError on a
    decidable mismatch or on logits outside rel_tol * max(1, |ref|_inf)."""
    rep = rep if rep is not None else StepReport()
    B, n, D = len(states), len(tmpl), ref.cfg.draft_heads
    Ls = [st.length for st in ref_states]
    out = be.step_tree(states, tmpl, k, prune, trace=True)
    tr = out.trace
    parent = np.asarray(tmpl.parent, dtype=np.int64)
    depth = np.asarray(tmpl.depth, dtype=np.int64)
    mask = tmpl.mask()
    Pn = len(tmpl.parent_nodes)
    row_base = 0
    for b in range(B):
        sr, L = ref_states[b], Ls[b]
        # -- draft heads on the last committed row: rank-wise, where the oracle's score gaps are decidable
        hid = sr.last_hidden
        dtok, dval = tr["draft_tokens"][b], tr["draft_val"][b]
        for d in range(D):
            lg = hid @ ref.w["w_draft"][d]
            _note_err(rep, "draft", dval[d], lg[dtok[d]])
        e_draft = 2 * max(rep.err["draft"], 1e-3)
        for d in range(D):
            lg = hid @ ref.w["w_draft"][d]
            order = np.argsort(-lg, kind="stable")
            s = lg[order[: k + 1]]
            # every device pick is the oracle's r-th best within the error bound (no rank is skipped) ...
            assert np.all(lg[dtok[d]] >= s[:k] - e_draft) and len(set(dtok[d].tolist())) == k, ("draft", b, d)
            # ... and is the oracle's r-th token wherever the neighbouring score gaps exceed it
            for r in range(k):
                ok = (r == 0 or s[r - 1] - s[r] > e_draft) and (r + 1 >= s.size or s[r] - s[r + 1] > e_draft)
                rep.count("draft", ok, 1)
                if ok:
                    assert int(dtok[d, r]) == int(order[r]), ("draft", b, d, r, int(dtok[d, r]), int(order[r]))
        # -- root (argmax of the last committed row): decided by the oracle's top-2 gap
        root_ref = int(np.argmax(sr.last_logits))
        root_dev = int(tr["root"][b])
        # -- the tree of the device's drafts; the device's survivors fed to the oracle's prune callback
        tokens = tr["tokens"][b].astype(np.int64)
        assert np.array_equal(tokens, dtok[depth - 1, np.asarray(tmpl.rank) - 1]), "K1 tree tokens"
        positions = L + depth - 1
        assert np.array_equal(tr["positions"][b], positions), "K1 positions"
        alive = tr["alive"][b].astype(bool)
        surv = [int(i) for i in np.flatnonzero(alive)]
        kw = {}
        cb = None
        if prune is not None:
            cb = _Replay(surv)
            kw = dict(prune_layer=prune.layer, early_topk=prune.topk, prune_callback=cb)
        fwd = ref.forward_tree(sr, tokens, positions, mask, **kw)
        assert list(fwd.survivors) == surv
        if prune is not None and Pn > 0:
            # -- K3 membership: child survives iff its token ranks < K in the parent's early row
            early_ref = cb.early[tmpl.parent_nodes]  # [Pn, V]
            early_dev = tr["early"][b * Pn:(b + 1) * Pn]
            _note_err(rep, "early", early_dev, early_ref)
            e_early = 2 * max(rep.err["early"], 1e-3)
            K = min(prune.topk, ref.cfg.vocab)
            member_ref = np.ones(n, dtype=bool)
            decid = np.ones(n, dtype=bool)
            for j, pnode in enumerate(tmpl.parent_nodes):
                row = early_ref[j]
                srt = np.sort(row)[::-1]
                vK, vK1 = srt[K - 1], (srt[K] if K < srt.size else -np.inf)
                for i in np.flatnonzero(parent == pnode):
                    order_row = np.argsort(-row, kind="stable")[:K]
                    member_ref[i] = tokens[i] in set(order_row.tolist())
                    decid[i] = (row[tokens[i]] - vK1 > e_early) if member_ref[i] else (vK - row[tokens[i]] > e_early)
            alive_ref = np.zeros(n, dtype=bool)
            path_ok = np.zeros(n, dtype=bool)
            for i in range(n):
                p = parent[i]
                alive_ref[i] = member_ref[i] and (p < 0 or alive_ref[p])
                path_ok[i] = decid[i] and (p < 0 or path_ok[p])
            rep.count("member", path_ok.sum(), n)
            assert np.array_equal(alive[path_ok], alive_ref[path_ok]), ("survivors", b)
        # -- logits of every surviving row, then argmax where decidable
        rows = tr["node_row"][b][np.asarray(surv, dtype=np.int64)]
        lg_dev = tr["row_logits"][rows]
        _note_err(rep, "logits", lg_dev, fwd.logits)
        bound = rel_tol * max(1.0, rep.scale["logits"])
        assert rep.err["logits"] <= bound, ("logits", rep.err["logits"], bound)
        e_lg = 2 * max(rep.err["logits"], 1e-3)
        gap = _top2_gap(fwd.logits)
        am_dev = tr["row_argmax"][rows]
        decid_rows = gap > e_lg
        rep.count("argmax", decid_rows.sum(), len(rows))
        assert np.array_equal(am_dev[decid_rows], fwd.argmax[decid_rows]), ("row argmax", b)
        root_ok = float(_top2_gap(sr.last_logits)) > e_lg
        rep.count("root", root_ok, 1)
        if root_ok:
            assert root_dev == root_ref, ("root", b, root_dev, root_ref)
        # -- greedy walk on the pruned tree: equal when every decision it reads is decidable
        sub = op.restrict(op.Tree(tuple(op.Node(int(tokens[i]), int(parent[i]), int(depth[i]), int(tmpl.rank[i]))
                                        for i in range(n)), root_dev), surv)
        acc_ref, bonus_ref = op.verify(sub, fwd.argmax, root_ref)
        a = int(out.acc_len[b])
        acc_dev = [int(v) for v in out.acc_surv[b, :a]]
        bonus_dev = int(out.committed[b, a])
        walk_ok = root_ok and all(decid_rows[j] for j in acc_ref)
        rep.count("walk", walk_ok, 1)
        if walk_ok:
            assert (tuple(acc_dev), bonus_dev) == (tuple(acc_ref), bonus_ref), ("walk", b, acc_dev, acc_ref)
        # device walk consistency with its own row argmax (always exact)
        acc_self, bonus_self = op.verify(sub, am_dev, root_dev)
        assert (tuple(acc_dev), bonus_dev) == (tuple(acc_self), bonus_self), ("K5 walk", b)
        committed = [int(t) for t in out.committed[b, : a + 1]]
        assert committed == [int(tokens[surv[j]]) for j in acc_dev] + [bonus_dev]
        rep.accepted += a
        # -- teacher forcing: the oracle commits what the device committed
        ref.commit(sr, acc_dev, bonus_dev)
        row_base += len(surv)
    return rep
