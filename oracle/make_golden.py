"""TEST INFRASTRUCTURE ONLY: generate tests/golden/ from the REAL reference.

Run in the build container (where /root/reference exists):

    python oracle/make_golden.py

It imports the unmodified reference package `treedecode` from
/root/reference/pkg/src (read-only), drives it through its own public API
(DecodeEngine, TinyTransformer, config builders) and writes small fixtures:

  tests/golden/run_tiny_<mode>.json   configs/run_tiny.json in every engine mode:
                                      prompts, transcripts, metrics.jsonl records,
                                      summary, plan events (simulated clock)
  tests/golden/run_tiny_trace.json    per-sequence step records of the propd_full
                                      run (tree tokens/positions, early top-K lists,
                                      survivors, argmax, accepted, bonus)
  tests/golden/c1_ar.json             greedy AR transcripts for the acceptance-gate
                                      C1 model (TinyTransformer seed 17) + prompts
  tests/golden/forward_cases.npz      forward_tree logits (fp64) for random trees,
                                      pruned and unpruned, on two model configs
  tests/golden/cli_run_tiny/          the reference CLI's run outputs for configs/run_tiny.json
                                      (transcripts, metrics.jsonl, summary.csv, plan_events.jsonl)
  tests/golden/cli_sweep_tiny/        the reference CLI's sweep.csv (mode x batch)
  tests/golden/gate_numbers.json      worked-number anchors (mask text, verify walks,
                                      prune cases, selection curves)
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
REF_PKG = Path("/root/reference/pkg")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def main() -> None:
    sys.path.insert(0, str(REF_SRC))
    import treedecode  # noqa: F401  (the reference, unmodified)
    from treedecode import config as tcfg
    from treedecode.acceptance import AcceptanceStats, HeadPredictions, grid_candidates, select_best_nodes
    from treedecode.backends import TinyTransformer, TinyTransformerConfig
    from treedecode.engine import MODES, DecodeEngine
    from treedecode.pruning import PruneConfig, prune
    from treedecode.token_tree import build_tree, complete_tree_paths, format_mask, make_mask
    from treedecode.verification import verify

    OUT.mkdir(parents=True, exist_ok=True)

    # 1. run_tiny in every mode --------------------------------------------
    base = tcfg.load_config(REF_PKG / "configs" / "run_tiny.json")
    for mode in MODES:
        cfg = json.loads(json.dumps(base))
        cfg["engine"]["mode"] = mode
        backend = tcfg.build_backend(cfg)
        engine = DecodeEngine(backend, tcfg.build_engine_config(cfg), tcfg.build_latency(cfg))
        prompts = tcfg.build_prompts(cfg, backend.vocab_size)
        res = engine.run(prompts, cfg["workload"]["max_tokens"], batch_size=cfg["workload"]["batch_size"])
        s = res.summary
        doc = {
            "mode": mode,
            "prompts": res.prompts,
            "transcripts": res.transcripts,
            "metrics": [m.to_json() for m in res.metrics],
            "summary": {k: getattr(s, k) for k in ("mode", "iterations", "total_tokens", "total_time",
                                                  "tokens_per_sec", "mean_accepted", "mean_prune_rate",
                                                  "mean_tree_size")},
            "plan_events": [
                {"iteration": e.iteration, "trigger": e.trigger, "chosen_size": e.chosen_size,
                 "l_curve": {str(k): v for k, v in e.l_curve.items()},
                 "v_curve": {str(k): v for k, v in e.v_curve.items()}}
                for e in res.plan_events
            ],
            "final_P": engine.stats.P.tolist(),
        }
        (OUT / f"run_tiny_{mode}.json").write_text(json.dumps(doc))
        if mode == "propd_full":
            shipped = [(REF_PKG / "out" / "run_tiny" / f"transcript_{i:03d}.txt").read_text()
                       for i in range(len(res.prompts))]
            mine = [" ".join(map(str, p)) + "\n" + " ".join(map(str, t)) + "\n"
                    for p, t in zip(res.prompts, res.transcripts)]
            assert shipped == mine, "reference no longer reproduces its shipped run_tiny outputs"

    # 2. step trace of the propd_full run -----------------------------------
    cfg = json.loads(json.dumps(base))
    trace: list = []

    class Recorder(TinyTransformer):
        def draft(self, state, k):
            out = super().draft(state, k)
            state._rec_draft = out.tokens.tolist()
            return out

        def forward_tree(self, state, tokens, positions, mask, *, prune_layer=None, early_topk=0,
                         prune_callback=None):
            rec = {"length": state.length, "tokens": [int(t) for t in tokens],
                   "positions": [int(p) for p in positions], "draft_tokens": state._rec_draft,
                   "root": int(np.argmax(state.last_logits))}
            cb = prune_callback
            if cb is not None:
                def cb(lists, _inner=prune_callback, _rec=rec):
                    _rec["early_lists"] = [list(map(int, r)) for r in lists]
                    return _inner(lists)
            fwd = super().forward_tree(state, tokens, positions, mask, prune_layer=prune_layer,
                                       early_topk=early_topk, prune_callback=cb)
            rec["survivors"] = list(fwd.survivors)
            rec["argmax"] = [int(a) for a in fwd.argmax]
            self._rec = rec
            return fwd

        def commit(self, state, accepted, bonus):
            if getattr(self, "_rec", None) is not None:
                self._rec["accepted"] = [int(a) for a in accepted]
                self._rec["bonus"] = int(bonus)
                trace.append(self._rec)
                self._rec = None
            super().commit(state, accepted, bonus)

    b = cfg["backend"]
    backend = Recorder(TinyTransformerConfig(seed=b["seed"], **b["tiny"]))
    engine = DecodeEngine(backend, tcfg.build_engine_config(cfg), tcfg.build_latency(cfg))
    prompts = tcfg.build_prompts(cfg, backend.vocab_size)
    engine.run(prompts, cfg["workload"]["max_tokens"], batch_size=cfg["workload"]["batch_size"])
    (OUT / "run_tiny_trace.json").write_text(json.dumps({"records": trace}))

    # 3. C1 greedy AR transcripts (tests/test_acceptance.py:47-49, 80-83) ----
    c1 = TinyTransformerConfig(layers=4, hidden=64, heads=4, vocab=256, draft_heads=4, max_positions=64, seed=17)
    tt = TinyTransformer(c1)
    rng = np.random.default_rng(101)
    c1_prompts = [rng.integers(0, c1.vocab, size=8).tolist() for _ in range(200)]
    ar = []
    for p in c1_prompts:
        st = tt.prefill(p)
        out = []
        for _ in range(10):
            tok = tt.next_argmax(st)
            tt.commit(st, [], tok)
            out.append(int(tok))
        ar.append(out)
    (OUT / "c1_ar.json").write_text(json.dumps({"prompts": c1_prompts, "transcripts": ar, "max_tokens": 10}))

    # 4. forward_tree logits on random trees --------------------------------
    arrays = {}
    meta = []
    cases = [("c2", c1), ("tb", TinyTransformerConfig(layers=3, hidden=32, heads=2, vocab=64, draft_heads=3,
                                                        max_positions=96, seed=5))]
    for tag, mcfg in cases:
        model = TinyTransformer(mcfg)
        g = np.random.default_rng(2024)
        for case in range(8):
            depth, k = 3, 3
            universe = complete_tree_paths(depth, k)
            sel = set()
            for p in sorted(universe, key=len):
                if (len(p) == 1 or p[:-1] in sel) and g.random() < 0.6:
                    sel.add(p)
            if not sel:
                sel.add((1,))
            grid = g.choice(mcfg.vocab, size=depth * k, replace=False).reshape(depth, k)
            preds = HeadPredictions(grid.astype(np.int64), -np.tile(np.arange(k, dtype=np.float64), (depth, 1)))
            tree = build_tree(preds, sel, root_token=0)
            ctx = g.integers(0, mcfg.vocab, size=int(g.integers(3, 9))).tolist()
            mask = make_mask(tree)
            positions = len(ctx) + tree.depths - 1
            st = model.prefill(ctx)
            pl = 2 if case % 2 else None
            if pl is not None:
                keep = []
                kept = set()
                for i, nd in enumerate(tree.nodes):
                    if (nd.parent == -1 or nd.parent in kept) and g.random() < 0.7:
                        keep.append(i)
                        kept.add(i)
                if not keep:
                    keep = [0]
                box = {}

                def cb(lists, _keep=keep, _box=box):
                    _box["lists"] = lists
                    return _keep

                fwd = model.forward_tree(st, tree.tokens, positions, mask, prune_layer=pl, early_topk=5,
                                         prune_callback=cb)
                arrays[f"{tag}_{case}_early"] = np.asarray(box["lists"], dtype=np.int64)
            else:
                fwd = model.forward_tree(st, tree.tokens, positions, mask)
            key = f"{tag}_{case}"
            arrays[key + "_logits"] = fwd.logits
            arrays[key + "_tokens"] = tree.tokens
            arrays[key + "_positions"] = positions
            arrays[key + "_mask"] = mask
            arrays[key + "_ctx"] = np.asarray(ctx, dtype=np.int64)
            arrays[key + "_survivors"] = np.asarray(fwd.survivors, dtype=np.int64)
            arrays[key + "_last_logits"] = st.last_logits
            arrays[key + "_last_hidden"] = st.last_hidden
            meta.append({"key": key, "model": mcfg.__dict__, "prune_layer": pl})
    np.savez_compressed(OUT / "forward_cases.npz", **arrays)
    (OUT / "forward_cases.json").write_text(json.dumps(meta))

    # 5. worked-number anchors ---------------------------------------------
    def preds_from(grid):
        t = np.asarray(grid, dtype=np.int64)
        return HeadPredictions(t, -np.tile(np.arange(t.shape[1], dtype=np.float64), (t.shape[0], 1)))

    fig = build_tree(preds_from([[10, 11], [20, 21], [30, 31]]), {(1,), (1, 1), (1, 2), (1, 1, 1)}, root_token=5)
    walks = []
    for root, am in [(10, [20, 30, 99, 77]), (10, [21, 0, 55, 0]), (404, [1, 2, 3, 4]), (10, [22, 9, 9, 9])]:
        r = verify(fig, am, root)
        walks.append({"root": root, "argmax": am, "accepted": list(r.accepted), "bonus": r.bonus})
    chain = build_tree(preds_from([[1], [3], [5]]), {(1,), (1, 1), (1, 1, 1)}, root_token=0)
    prunes = []
    for lists in ([[3, 99], [98, 97], [96]], [[99], [5], []], [[3], [5], []]):
        d = prune(chain, lists, PruneConfig(layer=2, topk=2))
        prunes.append({"lists": lists, "survivors": list(d.survivors), "rate": d.prune_rate})
    sel_cases = []
    g = np.random.default_rng(77)
    for D, K in [(2, 2), (3, 3), (4, 3), (4, 16), (4, 64)]:
        st = AcceptanceStats(D, K, alpha=0.05)
        if (D, K) != (4, 3):
            st.P = np.sort(g.uniform(0.0, 1.0, size=(D, K)), axis=1)
        out = select_best_nodes(st, list(range(1, D * K + 1)))
        sel_cases.append({"D": D, "K": K, "P": st.P.tolist(),
                          "order": [list(p) for p in out[D * K].paths],
                          "l": [out[s].expected_length for s in range(1, D * K + 1)]})
    gate = {"fig_mask": format_mask(make_mask(fig)), "walks": walks, "prunes": prunes,
            "selections": sel_cases, "grid_4_3": [list(p) for p in grid_candidates(4, 3)]}
    (OUT / "gate_numbers.json").write_text(json.dumps(gate))

    # 6. the reference CLI's own output files (cli.py:27-73) -------------------
    import shutil

    from treedecode import cli as tcli

    cli_dir = OUT / "cli_run_tiny"
    shutil.rmtree(cli_dir, ignore_errors=True)
    shutil.copy(REF_PKG / "configs" / "run_tiny.json", OUT / "run_tiny_config.json")
    assert tcli.main(["run", "--config", str(OUT / "run_tiny_config.json"), "--out-dir", str(cli_dir),
                      "--verbose"]) == 0
    sweep_cfg = json.loads((REF_PKG / "configs" / "run_tiny.json").read_text())
    sweep_cfg["sweep"] = {"mode": ["static_tree", "propd_full"], "batch": [2, 4]}
    (OUT / "sweep_tiny_config.json").write_text(json.dumps(sweep_cfg, indent=2))
    assert tcli.main(["sweep", "--config", str(OUT / "sweep_tiny_config.json"), "--axis", "mode", "--axis", "batch",
                      "--out-dir", str(OUT / "cli_sweep_tiny")]) == 0
    print(f"golden fixtures written to {OUT}")


if __name__ == "__main__":
    main()
