"""TEST INFRASTRUCTURE: a CPU stand-in for B200Backend's batched API, built
on the oracle (oracle/treedecode_port.py).  It lets the CPU suite drive the
product DecodeEngine's control flow — planning, sharding across gloo ranks,
acceptance-record gathering and ordered replay — without a GPU.  It is never
used by the product."""

from __future__ import annotations

from types import SimpleNamespace

import numpy as np
import torch

from oracle import treedecode_port as op


class OracleBatchBackend:
    def __init__(self, cfg: op.TinyCfg):
        self.model = op.TinyModel(cfg)
        self.cfg = cfg
        self.device = torch.device("cpu")
        self.torch = torch

    vocab_size = property(lambda self: self.cfg.vocab)
    num_layers = property(lambda self: self.cfg.layers)
    draft_head_count = property(lambda self: self.cfg.draft_heads)

    def prefill_batch(self, prompts):
        return [self.model.prefill(p) for p in prompts]

    def release(self, state):
        pass

    def step_autoregressive(self, states):
        out = []
        for st in states:
            tok = self.model.next_argmax(st)
            self.model.commit(st, [], tok)
            out.append(tok)
        return np.array(out)

    def step_tree(self, states, tmpl, k, prune=None, trace=False, stats=None, accept=None):
        D = self.cfg.draft_heads
        B = len(states)
        committed = np.full((B, D + 1), -1, dtype=np.int32)
        acc_len = np.zeros(B, dtype=np.int32)
        acc_surv = np.full((B, D), -1, dtype=np.int32)
        surv_cnt = np.zeros(B, dtype=np.int32)
        ranks = np.zeros((B, D), dtype=np.int8)
        for b, st in enumerate(states):
            pred = self.model.draft(st, k)
            root = self.model.next_argmax(st)
            tree = op.build_tree(pred, tmpl.paths, root_token=0)
            mask = op.make_mask(tree)
            pos = st.length + tree.depths - 1
            if prune is not None:
                box = {}

                def cb(lists, _t=tree, _b=box):
                    _b["s"] = op.prune(_t, lists, op.PruneCfg(prune.layer, prune.topk))[0]
                    return _b["s"]

                fwd = self.model.forward_tree(st, tree.tokens, pos, mask, prune_layer=prune.layer,
                                              early_topk=prune.topk, prune_callback=cb)
                vtree = op.restrict(tree, box["s"])
            else:
                fwd = self.model.forward_tree(st, tree.tokens, pos, mask)
                vtree = tree
            acc, bonus = op.verify(vtree, fwd.argmax, root)
            self.model.commit(st, acc, bonus)
            newly = [vtree.nodes[i].token for i in acc] + [bonus]
            committed[b, : len(newly)] = newly
            acc_len[b] = len(acc)
            acc_surv[b, : len(acc)] = acc
            surv_cnt[b] = len(fwd.survivors)
            for d in range(min(len(newly), D)):
                r = pred.rank_of(d + 1, newly[d])
                ranks[b, d] = r if r is not None else -1
        out = SimpleNamespace(committed=committed, acc_len=acc_len, acc_surv=acc_surv, surv_cnt=surv_cnt,
                              ranks_dev=torch.from_numpy(ranks), ranks=ranks, trace=None, order=None, lcurve=None)
        if stats is not None:
            P, counts, alpha, order, lcurve = stats
            self.stats_replay_select(out.ranks_dev, B, P, counts, alpha, order, lcurve)
            out.order, out.lcurve = order.numpy().copy(), lcurve.numpy().copy()
        return out

    def stats_replay_select(self, ranks, S, P, counts, alpha, order, lcurve):
        """Host restatement of propd_stats_replay_select (acceptance.py:96-113, 186-206)."""
        D, k = P.shape
        st = op.Stats(D, k, alpha=alpha)
        st.P = P.numpy().copy()
        st.counts = counts.numpy().copy()
        toks = np.arange(D * k).reshape(D, k)
        preds = op.Preds(toks, -np.tile(np.arange(float(k)), (D, 1)))
        for s in range(S):
            realized = {}
            for d in range(D):
                r = int(ranks[s, d])
                if r == 0:
                    continue
                realized[d + 1] = int(toks[d, r - 1]) if r > 0 else -7
            st.update(realized, preds)
        P.copy_(torch.from_numpy(st.P))
        counts.copy_(torch.from_numpy(st.counts))
        sel = op.select_best_nodes(st, list(range(1, D * k + 1)))
        uni = op.grid_candidates(D, k)
        idx = {p: i for i, p in enumerate(uni)}
        order.copy_(torch.tensor([idx[p] for p in sel[D * k][0]], dtype=torch.int32))
        lcurve.copy_(torch.tensor([sel[s][1] for s in range(1, D * k + 1)], dtype=torch.float64))
