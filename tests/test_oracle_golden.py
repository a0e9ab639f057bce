"""Pin the CPU oracle (oracle/treedecode_port.py) to outputs of the real
reference (tests/golden/, made by oracle/make_golden.py).  CPU only."""

import json
import os

import numpy as np
import pytest

from oracle import treedecode_port as op

MODES = op.MODES


def load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as fh:
        return json.load(fh)


def run_tiny(mode, trace=None):
    cfg = op.RUN_TINY
    ecfg = op.EngineCfg(**{**cfg["engine"].__dict__, "mode": mode})
    model = op.TinyModel(cfg["model"])
    eng = op.Engine(model, ecfg, op.Clock(**cfg["clock"]), trace=trace)
    w = cfg["workload"]
    prompts = op.synthetic_prompts(model.vocab_size, w["num_prompts"], w["prompt_len"], w["seed"])
    return eng, eng.run(prompts, w["max_tokens"], batch_size=w["batch_size"])


@pytest.mark.parametrize("mode", MODES)
def test_run_tiny_all_modes_byte_identical(golden_dir, mode):
    g = load(golden_dir, f"run_tiny_{mode}.json")
    eng, res = run_tiny(mode)
    assert res["prompts"] == g["prompts"]
    assert res["transcripts"] == g["transcripts"]
    # metrics.jsonl records compare exactly, floats included (simulated clock)
    assert [json.dumps(m) for m in res["metrics"]] == [json.dumps(m) for m in g["metrics"]]
    assert res["summary"] == g["summary"]
    assert np.array_equal(eng.stats.P, np.array(g["final_P"]))
    ev = [{**e, "l_curve": {str(k): v for k, v in e["l_curve"].items()},
           "v_curve": {str(k): v for k, v in e["v_curve"].items()}} for e in res["plan_events"]]
    assert ev == g["plan_events"]


def test_step_trace_matches_reference(golden_dir):
    g = load(golden_dir, "run_tiny_trace.json")["records"]
    mine = []
    run_tiny("propd_full", trace=lambda it, rec: mine.append(rec))
    assert len(mine) == len(g)
    for a, b in zip(mine, g):
        for key in ("tokens", "positions", "survivors", "argmax", "accepted", "bonus", "early_lists",
                    "draft_tokens", "root", "length"):
            assert a[key] == b[key], key


def test_c1_ar_transcripts(golden_dir):
    g = load(golden_dir, "c1_ar.json")
    model = op.TinyModel(op.TinyCfg(layers=4, hidden=64, heads=4, vocab=256, draft_heads=4,
                                    max_positions=64, seed=17))
    for p, t in list(zip(g["prompts"], g["transcripts"]))[:40]:
        assert op.greedy_transcript(model, p, g["max_tokens"]) == t


def test_forward_cases_logits(golden_dir):
    meta = load(golden_dir, "forward_cases.json")
    arr = np.load(os.path.join(golden_dir, "forward_cases.npz"))
    models = {}
    for m in meta:
        key = m["key"]
        mc = op.TinyCfg(**m["model"])
        model = models.setdefault(key.split("_")[0], op.TinyModel(mc))
        st = model.prefill(arr[key + "_ctx"].tolist())
        np.testing.assert_allclose(st.last_logits, arr[key + "_last_logits"], rtol=1e-12, atol=1e-13)
        surv = arr[key + "_survivors"].tolist()
        kw = {}
        if m["prune_layer"] is not None:
            box = {}

            def cb(lists, _s=surv, _b=box):
                _b["lists"] = lists
                return _s

            kw = dict(prune_layer=m["prune_layer"], early_topk=5, prune_callback=cb)
        fwd = model.forward_tree(st, arr[key + "_tokens"], arr[key + "_positions"], arr[key + "_mask"], **kw)
        assert list(fwd.survivors) == surv
        np.testing.assert_allclose(fwd.logits, arr[key + "_logits"], rtol=1e-12, atol=1e-13)
        if kw:
            assert np.array_equal(np.asarray(box["lists"]), arr[key + "_early"])


def test_gate_numbers(golden_dir):
    g = load(golden_dir, "gate_numbers.json")

    def preds_from(grid):
        t = np.asarray(grid, dtype=np.int64)
        return op.Preds(t, -np.tile(np.arange(t.shape[1], dtype=np.float64), (t.shape[0], 1)))

    fig = op.build_tree(preds_from([[10, 11], [20, 21], [30, 31]]), {(1,), (1, 1), (1, 2), (1, 1, 1)},
                        root_token=5)
    assert op.format_mask(op.make_mask(fig)) == g["fig_mask"]
    for w in g["walks"]:
        acc, bonus = op.verify(fig, w["argmax"], w["root"])
        assert list(acc) == w["accepted"] and bonus == w["bonus"]
    chain = op.build_tree(preds_from([[1], [3], [5]]), {(1,), (1, 1), (1, 1, 1)}, root_token=0)
    for p in g["prunes"]:
        surv, rate = op.prune(chain, p["lists"], op.PruneCfg(layer=2, topk=2))
        assert list(surv) == p["survivors"] and rate == p["rate"]
    for c in g["selections"]:
        st = op.Stats(c["D"], c["K"], alpha=0.05)
        st.P = np.array(c["P"])
        out = op.select_best_nodes(st, list(range(1, c["D"] * c["K"] + 1)))
        assert [list(p) for p in out[c["D"] * c["K"]][0]] == c["order"]
        assert [out[s][1] for s in range(1, c["D"] * c["K"] + 1)] == c["l"]
    assert [list(p) for p in op.grid_candidates(4, 3)] == g["grid_4_3"]
