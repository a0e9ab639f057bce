"""End-to-end parity of the B200 decode path (fp32 parity mode) with the
reference, through golden fixtures of the real reference and the CPU oracle.

Bar: bit-exact transcripts, per-iteration metrics (simulated clock), plan
events, tree tokens/positions, survivor sets, accepted indices, bonus tokens
and the fp64 acceptance statistics; logits within
  max |err| <= 2e-5 * max(1, |ref|_inf)   (fp32 vs the reference's fp64).
"""

import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import treedecode_port as op  # noqa: E402
from paper_2402_13485_b200 import (B200Backend, DecodeEngine, EngineConfig, PruneConfig,  # noqa: E402
                                   SchedulerConfig, TinyTransformerConfig)
from paper_2402_13485_b200.tree import TreeTemplate  # noqa: E402

MODES = op.MODES
RUN_TINY = op.RUN_TINY


def load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as fh:
        return json.load(fh)


def product_cfg(ecfg: op.EngineCfg, mode: str) -> EngineConfig:
    s = ecfg.scheduler
    return EngineConfig(mode=mode, draft_heads=ecfg.draft_heads, draft_topk=ecfg.draft_topk,
                        prune=PruneConfig(ecfg.prune.layer, ecfg.prune.topk) if ecfg.prune else None,
                        scheduler=SchedulerConfig(s.resize_batch_delta, s.resize_seqlen_delta, s.replan_period,
                                                  s.size_candidates),
                        acceptance_alpha=ecfg.acceptance_alpha)


def tiny_backend(mc: op.TinyCfg, slots=8, **kw):
    return B200Backend(TinyTransformerConfig(**mc.__dict__), dtype="fp32", max_slots=slots, **kw)


@pytest.fixture(scope="module")
def run_tiny_backend():
    return tiny_backend(RUN_TINY["model"])


@pytest.fixture(scope="module")
def run_tiny_graph_backend():
    return tiny_backend(RUN_TINY["model"], use_graphs=True)


@pytest.mark.parametrize("graphs", [False, True])
@pytest.mark.parametrize("mode", MODES)
def test_run_tiny_batched_engine_matches_reference(golden_dir, run_tiny_backend, run_tiny_graph_backend, mode,
                                                   graphs):
    g = load(golden_dir, f"run_tiny_{mode}.json")
    be = run_tiny_graph_backend if graphs else run_tiny_backend
    eng = DecodeEngine(be, product_cfg(RUN_TINY["engine"], mode), op.Clock(**RUN_TINY["clock"]))
    w = RUN_TINY["workload"]
    res = eng.run(g["prompts"], w["max_tokens"], batch_size=w["batch_size"])
    assert res.transcripts == g["transcripts"]
    assert [json.dumps(m.to_json()) for m in res.metrics] == [json.dumps(m) for m in g["metrics"]]
    s = res.summary
    assert {k: getattr(s, k) for k in g["summary"]} == g["summary"]
    ev = [{"iteration": e.iteration, "trigger": e.trigger, "chosen_size": e.chosen_size,
           "l_curve": {str(k): v for k, v in e.l_curve.items()},
           "v_curve": {str(k): v for k, v in e.v_curve.items()}} for e in res.plan_events]
    assert ev == g["plan_events"]
    if mode != "autoregressive":
        assert np.array_equal(eng.stats_P, np.array(g["final_P"]))


def test_step_records_match_reference_trace(golden_dir, run_tiny_backend):
    g = load(golden_dir, "run_tiny_trace.json")["records"]
    mine = []
    eng = DecodeEngine(run_tiny_backend, product_cfg(RUN_TINY["engine"], "propd_full"),
                       op.Clock(**RUN_TINY["clock"]), trace=lambda it, rec: mine.append(rec))
    w = RUN_TINY["workload"]
    prompts = op.synthetic_prompts(256, w["num_prompts"], w["prompt_len"], w["seed"])
    eng.run(prompts, w["max_tokens"], batch_size=w["batch_size"])
    assert len(mine) == len(g)
    for a, b in zip(mine, g):
        for key in ("tokens", "positions", "draft_tokens", "root", "survivors", "argmax", "accepted", "bonus"):
            assert a[key] == b[key], key


@pytest.mark.parametrize("mode", MODES)
def test_per_sequence_plugin_api_in_reference_loop(golden_dir, mode):
    """The oracle's restatement of the reference DecodeEngine driving
    B200Backend through the per-sequence ModelBackend API (drop-in path)."""
    g = load(golden_dir, f"run_tiny_{mode}.json")
    be = tiny_backend(RUN_TINY["model"], slots=12)
    ecfg = op.EngineCfg(**{**RUN_TINY["engine"].__dict__, "mode": mode})
    eng = op.Engine(be, ecfg, op.Clock(**RUN_TINY["clock"]))
    w = RUN_TINY["workload"]
    res = eng.run(g["prompts"], w["max_tokens"], batch_size=w["batch_size"])
    assert res["transcripts"] == g["transcripts"]
    assert [json.dumps(m) for m in res["metrics"]] == [json.dumps(m) for m in g["metrics"]]


def test_c1_losslessness_all_tree_modes(golden_dir):
    """Acceptance-gate C1 (tests/test_acceptance.py:77-121): every tree mode
    emits the greedy AR stream, 200 prompts, batch 25."""
    g = load(golden_dir, "c1_ar.json")
    mc = op.TinyCfg(layers=4, hidden=64, heads=4, vocab=256, draft_heads=4, max_positions=64, seed=17)
    be = tiny_backend(mc, slots=32)
    sched = SchedulerConfig(replan_period=8, size_candidates=(1, 2, 4, 6, 8))
    for mode in ("autoregressive", "static_tree", "prune_only", "dynamic_only", "propd_full"):
        cfg = EngineConfig(mode=mode, draft_heads=4, draft_topk=3, scheduler=sched, acceptance_alpha=None,
                           prune=PruneConfig(layer=2, topk=16) if mode in ("prune_only", "propd_full") else None)
        res = DecodeEngine(be, cfg, op.Clock()).run(g["prompts"], g["max_tokens"], batch_size=25)
        assert res.transcripts == g["transcripts"], mode


def test_forward_tree_logits_and_early_lists(golden_dir):
    meta = load(golden_dir, "forward_cases.json")
    arr = np.load(os.path.join(golden_dir, "forward_cases.npz"))
    backends = {}
    for m in meta:
        key = m["key"]
        tag = key.split("_")[0]
        if tag not in backends:
            backends[tag] = tiny_backend(op.TinyCfg(**m["model"]), slots=4)
        be = backends[tag]
        st = be.prefill(arr[key + "_ctx"].tolist())
        ref_last = arr[key + "_last_logits"]
        assert np.abs(be.last_logits_of(st) - ref_last).max() <= 2e-5 * max(1.0, np.abs(ref_last).max())
        surv = arr[key + "_survivors"].tolist()
        kw = {}
        box = {}
        if m["prune_layer"] is not None:
            def cb(lists, _s=surv, _b=box):
                _b["lists"] = lists
                return _s
            kw = dict(prune_layer=m["prune_layer"], early_topk=5, prune_callback=cb)
        fwd = be.forward_tree(st, arr[key + "_tokens"], arr[key + "_positions"], arr[key + "_mask"], **kw)
        ref = arr[key + "_logits"]
        assert list(fwd.survivors) == surv
        assert np.abs(fwd.logits - ref).max() <= 2e-5 * max(1.0, np.abs(ref).max())
        assert np.array_equal(fwd.argmax, np.argmax(ref, axis=1))
        if kw:
            assert np.array_equal(np.asarray(box["lists"]), arr[key + "_early"])


def test_plugin_api_errors_match_reference():
    be = tiny_backend(op.TinyCfg(layers=3, hidden=32, heads=2, vocab=64, draft_heads=3, max_positions=96, seed=5),
                      slots=4)
    with pytest.raises(ValueError, match="non-empty"):
        be.prefill([])
    with pytest.raises(ValueError, match="vocabulary"):
        be.prefill([0, 64])
    with pytest.raises(ValueError, match="max_positions"):
        be.prefill([0] * 97)
    st = be.prefill([3, 1, 4, 1])
    tmpl = TreeTemplate.from_paths([(1,), (2,), (1, 1)])
    toks = np.array([7, 9, 11])
    pos = 4 + tmpl.depth - 1
    mask = tmpl.mask()
    with pytest.raises(ValueError, match="sizes disagree"):
        be.forward_tree(st, toks, pos, mask[:-1])
    with pytest.raises(ValueError, match="follow the committed context"):
        be.forward_tree(st, toks, pos - 4, mask)
    with pytest.raises(ValueError, match="vocabulary"):
        be.forward_tree(st, toks + 64, pos, mask)
    cb = lambda lists: list(range(len(lists)))
    with pytest.raises(ValueError, match="strictly inside"):
        be.forward_tree(st, toks, pos, mask, prune_layer=3, early_topk=4, prune_callback=cb)
    with pytest.raises(ValueError, match="early_topk"):
        be.forward_tree(st, toks, pos, mask, prune_layer=1, early_topk=0, prune_callback=cb)
    with pytest.raises(ValueError, match="preceding tree forward"):
        be.commit(be.prefill([1, 2]), [0], 5)
    be.forward_tree(st, toks, pos, mask)
    with pytest.raises(ValueError, match="contiguous root chain"):
        be.commit(st, [0, 1], 0)
    be.commit(st, [0, 2], 42)
    assert st.committed == [3, 1, 4, 1, 7, 11, 42]
    fresh = be.prefill(st.committed)
    a, b = be.last_logits_of(st), be.last_logits_of(fresh)
    assert np.abs(a - b).max() <= 2e-5 * max(1.0, np.abs(b).max())
    with pytest.raises(ValueError):
        be.draft(st, 0)


def test_commit_equals_scratch_prefill_and_oracle():
    """commit (KV compaction) == scratch prefill == the fp64 oracle (tests/test_backends.py:140-155)."""
    mc = op.TinyCfg(layers=3, hidden=32, heads=2, vocab=64, draft_heads=3, max_positions=96, seed=5)
    be = tiny_backend(mc, slots=6)
    ref = op.TinyModel(mc)
    ctx = [3, 1, 4, 1, 5]
    st, rs = be.prefill(ctx), ref.prefill(ctx)
    rng = np.random.default_rng(0)
    for _ in range(6):
        pred = ref.draft(rs, 2)
        tree = op.build_tree(pred, op.complete_tree_paths(3, 2), root_token=0)
        mask = op.make_mask(tree)
        pos = rs.length + tree.depths - 1
        f1 = be.forward_tree(st, tree.tokens, pos, mask)
        f0 = ref.forward_tree(rs, tree.tokens, pos, mask)
        assert np.array_equal(f1.argmax, f0.argmax)
        acc, bonus = op.verify(tree, f0.argmax, ref.next_argmax(rs))
        if not acc and rng.random() < 0.7:  # force an accepted chain to exercise compaction
            acc = (0, 2)  # nodes (1,) -> (1, 1)
            bonus = int(f0.argmax[2])
        be.commit(st, list(acc), bonus)
        ref.commit(rs, list(acc), bonus)
        assert st.committed == rs.committed
        assert np.abs(be.last_logits_of(st) - rs.last_logits).max() <= 2e-5 * max(1.0, np.abs(rs.last_logits).max())
        assert be.next_argmax(st) == ref.next_argmax(rs)
        d1, d0 = be.draft(st, 2), ref.draft(rs, 2)
        assert np.array_equal(d1.tokens, d0.tokens)


def test_bf16_streaming_projections_match_cublas_path():
    """bf16 backend at 7B width (2 layers): the tcgen05 weight-streaming path
    (fused KV append / GELU / residual) vs the cuBLAS path.  Tolerance: final
    logits within 3e-2 * max(1, |ref|_inf) (bf16 rounding of different
    reduction orders)."""
    cfg = TinyTransformerConfig(layers=2, hidden=4096, heads=32, vocab=32000, draft_heads=4, max_positions=256, seed=1)
    a = B200Backend(cfg, dtype="bf16", random_device_init=True, max_slots=2, max_tree=16, use_gws=True)
    b = B200Backend(cfg, dtype="bf16", random_device_init=True, max_slots=2, max_tree=16, use_gws=False)
    prompt = list(range(100, 140))
    sa, sb = a.prefill(prompt), b.prefill(prompt)
    la, lb = a.last_logits_of(sa), b.last_logits_of(sb)
    assert np.abs(la - lb).max() <= 3e-2 * max(1.0, np.abs(lb).max())
    tmpl = TreeTemplate.from_paths(op.grid_candidates(4, 3))
    toks = np.arange(200, 200 + len(tmpl))
    pos = len(prompt) + tmpl.depth - 1
    fa = a.forward_tree(sa, toks, pos, tmpl.mask())
    fb = b.forward_tree(sb, toks, pos, tmpl.mask())
    assert np.abs(fa.logits - fb.logits).max() <= 3e-2 * max(1.0, np.abs(fb.logits).max())


def test_sync_free_post_prune_pass_matches_synced_pass():
    """bf16 at 7B width: the post-prune layers launched for the padded row
    capacity with the live row count read on the device (no mid-step sync)
    give the same survivors / accepted tokens as the synced pass sized on the
    host.  Structural outputs bit-exact; LM argmax of the surviving rows may
    differ only through fp32 reduction order (split-K atomics): >= 95% agree."""
    cfg = TinyTransformerConfig(layers=3, hidden=4096, heads=32, vocab=32000, draft_heads=4, max_positions=512, seed=2)
    tmpl = TreeTemplate.from_paths(op.grid_candidates(4, 3))
    outs = []
    for device_rows in (True, False):
        be = B200Backend(cfg, dtype="bf16", random_device_init=True, max_slots=3, max_tree=16)
        be.device_rows = device_rows
        states = be.synthetic_states(3, 200, seed=4)
        outs.append(be.step_tree(states, tmpl, 3, prune=PruneConfig(1, 50), trace=True))
        del be
    a, b = outs
    assert np.array_equal(a.trace["alive"], b.trace["alive"])
    assert np.array_equal(a.surv_cnt, b.surv_cnt)
    assert np.array_equal(a.trace["tokens"], b.trace["tokens"])
    alive = a.trace["alive"].astype(bool)
    ra = a.trace["row_argmax"][a.trace["node_row"][alive]]
    rb = b.trace["row_argmax"][b.trace["node_row"][alive]]
    assert (ra == rb).mean() >= 0.95
    if np.array_equal(ra, rb):
        assert np.array_equal(a.committed, b.committed) and np.array_equal(a.acc_len, b.acc_len)


def test_survivor_tier_variants_match_full_capacity_pass():
    """bf16 at 7B width, B=4 with a 64-node tree (256 pre-prune rows): the part-B variant chosen from the
    step's survivor-count read (<= 64 / 128 rows on the weight-streaming GEMMs, 32-row attention tiles
    when no sequence has more than 32 survivors) against the full-capacity variant (many-row GEMM, 64-row
    tiles).  Structural outputs bit-exact; argmax of the surviving rows >= 95% equal (fp32 reduction order
    differs between the two GEMM paths)."""
    cfg = TinyTransformerConfig(layers=3, hidden=4096, heads=32, vocab=32000, draft_heads=4, max_positions=512, seed=3)
    tmpl = TreeTemplate.from_paths(op.grid_candidates(4, 16))
    outs = []
    for split_sync in (True, False):
        be = B200Backend(cfg, dtype="bf16", random_device_init=True, max_slots=4, max_tree=64, use_graphs=True)
        be.ws_split_sync = split_sync
        states = be.synthetic_states(4, 300, seed=6)
        outs.append(be.step_tree(states, tmpl, 16, prune=PruneConfig(1, 50), trace=True))
        if split_sync:  # the tiered variants were captured up front
            assert sum(1 for key in be._graphs if key[0] == "B") >= 2
        del be
    a, b = outs
    assert np.array_equal(a.trace["alive"], b.trace["alive"])
    assert np.array_equal(a.surv_cnt, b.surv_cnt)
    alive = a.trace["alive"].astype(bool)
    ra = a.trace["row_argmax"][a.trace["node_row"][alive]]
    rb = b.trace["row_argmax"][b.trace["node_row"][alive]]
    assert (ra == rb).mean() >= 0.95
    if np.array_equal(ra, rb):
        assert np.array_equal(a.committed, b.committed) and np.array_equal(a.acc_len, b.acc_len)


@pytest.mark.parametrize("B,L,k", [(1, 1000, 16), (2, 37, 16), (4, 300, 16), (8, 200, 8)])
def test_qkv_tail_folded_into_attention_matches_tail_path(B, L, k):
    """bf16 at 7B width: tree passes whose QKV launch has no tail — the transposed attention reads Q and the
    tree rows' K/V from the fp32 accumulator and writes those K/V rows into the cache itself
    (PROPD_ATTN_QKV_F32) — against the QKV-tail path, pre-prune (64-node tree) and post-prune, ragged committed
    lengths (L - 13 b, one shorter than a key block).  Structural outputs bit-exact; the surviving tree rows'
    cache K/V within 2e-2 * max(1, |ref|_inf) (two runs: the split-K fp32 accumulation order differs, so bf16
    roundings may differ by an ulp); surviving rows' logits within 3e-2 * max(1, |ref|_inf) (the tail path may
    route latency-bound launches to the row-major kernel); argmax >= 95% equal."""
    cfg = TinyTransformerConfig(layers=3, hidden=4096, heads=32, vocab=32000, draft_heads=4, max_positions=1100,
                                seed=5)
    tmpl = TreeTemplate.from_paths(op.grid_candidates(4, k))
    outs, caches = [], []
    for fold in (True, False):
        be = B200Backend(cfg, dtype="bf16", random_device_init=True, max_slots=B, max_tree=64, use_graphs=True)
        be.ws_qkv_fold = fold
        states = be.synthetic_states(B, L, seed=9)
        for b, st in enumerate(states):  # ragged lengths
            Lb = max(1, L - 13 * b)
            be._len[st.slot] = Lb
            be.seq_len[st.slot] = Lb
            st.committed = st.committed[:Lb]
        lens = [be._len[st.slot] for st in states]
        outs.append(be.step_tree(states, tmpl, k, prune=PruneConfig(1, 50), trace=True))
        # tree rows of the last layer: cache slots L_b + node (before K5 compaction moved the accepted ones)
        caches.append([be.kcache[-1, st.slot, :, Lb + 1: Lb + len(tmpl)].float().cpu().numpy()
                       for st, Lb in zip(states, lens)])
        del be
    a, b = outs
    assert np.array_equal(a.trace["alive"], b.trace["alive"])
    assert np.array_equal(a.surv_cnt, b.surv_cnt)
    la, lb = a.trace["row_logits"], b.trace["row_logits"]
    assert np.abs(la - lb).max() <= 3e-2 * max(1.0, np.abs(lb).max())
    alive = a.trace["alive"].astype(bool)
    ra = a.trace["row_argmax"][a.trace["node_row"][alive]]
    rb = b.trace["row_argmax"][b.trace["node_row"][alive]]
    assert (ra == rb).mean() >= 0.95
    if np.array_equal(a.acc_len, b.acc_len) and not a.acc_len.any():  # nothing committed: rows stayed in place
        for ca, cb, al in zip(caches[0], caches[1], alive):
            keep = al[1:]  # surviving tree rows (node 0 is overwritten by the bonus row)
            assert keep.any() and np.abs(ca[:, keep] - cb[:, keep]).max() <= 2e-2 * max(1.0, np.abs(cb).max())


@pytest.mark.parametrize("mode", ["static_tree", "propd_full"])
def test_planted_acceptance_matches_oracle(mode):
    """Planted-acceptance harness: draft head 0 := the LM head on the same seeded weights for
    the B200 backend and the oracle, so every step accepts depth-1 nodes (multi-token commits, in-place KV
    compaction, acceptance statistics away from zero) — transcripts, metrics and P stay identical."""
    from paper_2402_13485_b200.weights import seeded_weights

    mc = op.TinyCfg(layers=4, hidden=64, heads=4, vocab=256, draft_heads=4, max_positions=160, seed=11)
    w = seeded_weights(TinyTransformerConfig(**mc.__dict__))
    w["w_draft"] = w["w_draft"].copy()
    w["w_draft"][0] = w["w_lm"]
    ecfg = op.EngineCfg(mode=mode, draft_heads=4, draft_topk=3, prune=op.PruneCfg(layer=2, topk=24),
                        scheduler=op.SchedCfg(replan_period=8, size_candidates=(1, 2, 4, 8, 12)))
    prompts = op.synthetic_prompts(256, 6, 7, 3)
    clock = dict(c0_base=3.0, c1_base=0.05, noise=0.02, seed=5)
    ref = op.Engine(op.TinyModel(mc, weights=w), ecfg, op.Clock(**clock)).run(prompts, 24, batch_size=3)
    be = B200Backend(TinyTransformerConfig(**mc.__dict__), dtype="fp32", max_slots=8, weights=w)
    res = DecodeEngine(be, product_cfg(ecfg, mode), op.Clock(**clock)).run(prompts, 24, batch_size=3)
    assert res.transcripts == ref["transcripts"]
    assert [m.to_json() for m in res.metrics] == ref["metrics"]
    assert res.summary.mean_accepted >= 0.9  # depth-1 accepted (almost) every step


def test_plant_draft_head_copies_lm_head():
    be = B200Backend(TinyTransformerConfig(layers=1, hidden=128, heads=1, vocab=512, draft_heads=3),
                     dtype="bf16", random_device_init=True, max_slots=2)
    be.plant_draft_head(1)
    assert torch.equal(be.w.w_draft[:, 512:1024], be.w.w_lm)
    with pytest.raises(ValueError, match="out of range"):
        be.plant_draft_head(3)


@pytest.mark.parametrize("threshold,acceptance", [(0.01, "greedy"), (None, "typical"), (0.02, "typical")])
def test_probability_prune_and_typical_acceptance_match_oracle(threshold, acceptance):
    """propd_full with probability-based pruning and/or typical acceptance on the device == the oracle engine
    with the same criteria (oracle probability_prune / typical_verify): transcripts and per-iteration metrics."""
    mc = op.TinyCfg(layers=4, hidden=64, heads=4, vocab=256, draft_heads=4, max_positions=160, seed=11)
    ecfg = op.EngineCfg(mode="propd_full", draft_heads=4, draft_topk=3,
                        prune=op.PruneCfg(layer=2, topk=24, threshold=threshold), acceptance=acceptance,
                        typical_epsilon=0.3, typical_alpha=0.5,
                        scheduler=op.SchedCfg(replan_period=8, size_candidates=(1, 2, 4, 8, 12)))
    prompts = op.synthetic_prompts(256, 6, 7, 3)
    clock = dict(c0_base=3.0, c1_base=0.05, noise=0.02, seed=5)
    ref = op.Engine(op.TinyModel(mc), ecfg, op.Clock(**clock)).run(prompts, 24, batch_size=3)
    pcfg = EngineConfig(mode="propd_full", draft_heads=4, draft_topk=3,
                        prune=PruneConfig(layer=2, topk=24, threshold=threshold),
                        scheduler=SchedulerConfig(replan_period=8, size_candidates=(1, 2, 4, 8, 12)),
                        acceptance=acceptance, typical_epsilon=0.3, typical_alpha=0.5)
    for graphs in (False, True):
        be = tiny_backend(mc, use_graphs=graphs)
        res = DecodeEngine(be, pcfg, op.Clock(**clock)).run(prompts, 24, batch_size=3)
        assert res.transcripts == ref["transcripts"]
        assert [m.to_json() for m in res.metrics] == ref["metrics"]
    if acceptance == "typical":
        assert ref["summary"]["mean_accepted"] > 0.3


@pytest.mark.parametrize("prune", [False, True])
def test_bf16_tree_pass_matches_fp64_oracle(prune):
    """bf16 performance mode vs the fp64 oracle on the same reference-initialised weights:
    dh = 128 heads so the tree pass runs the tcgen05 kernels (transposed attention for <= 64 rows, weight-
    streaming projections).  Logits within 5e-2 * max(1, |ref|_inf) (bf16 weights and activations vs fp64);
    argmax equal on every row whose oracle top-2 margin exceeds twice the measured max error (teacher-forced
    decisions; at least half the rows must be decidable so the check is not vacuous);
    survivors of the same prune decision identical."""
    mc = op.TinyCfg(layers=3, hidden=1024, heads=8, vocab=4096, draft_heads=2, max_positions=700, seed=3)
    ref = op.TinyModel(mc)
    be = B200Backend(TinyTransformerConfig(**mc.__dict__), dtype="bf16", max_slots=2, max_tree=64)
    rng = np.random.default_rng(9)
    prompt = rng.integers(0, mc.vocab, size=480).tolist()
    st_ref, st = ref.prefill(prompt), be.prefill(prompt)
    tmpl = TreeTemplate.from_paths(op.complete_tree_paths(2, 7)[:40])
    n = len(tmpl)
    tokens = rng.integers(0, mc.vocab, size=n)
    positions = len(prompt) + tmpl.depth.astype(np.int64) - 1
    mask = tmpl.mask()
    kw_ref, kw = {}, {}
    if prune:
        depth1 = {i for i in range(n) if tmpl.depth[i] == 1}
        keep = sorted(depth1 | {i for i in range(n) if tmpl.parent[i] in (0, 1) and i % 2 == 0})
        kw_ref = dict(prune_layer=1, early_topk=4, prune_callback=lambda lists: keep)
        kw = dict(prune_layer=1, early_topk=4, prune_callback=lambda lists: keep)
    fr = ref.forward_tree(st_ref, tokens, positions, mask, **kw_ref)
    fb = be.forward_tree(st, tokens, positions, mask, **kw)
    assert list(fb.survivors) == list(fr.survivors)
    scale = max(1.0, np.abs(fr.logits).max())
    bound = 5e-2 * scale
    err = np.abs(fb.logits - fr.logits).max()
    assert err <= bound, (err, bound)
    top2 = np.sort(fr.logits, axis=1)[:, -2:]
    decidable = (top2[:, 1] - top2[:, 0]) > 2 * max(err, 1e-3 * scale)
    assert np.array_equal(fb.argmax[decidable], fr.argmax[decidable])
    last_err = np.abs(be.last_logits_of(st) - st_ref.last_logits).max()
    assert last_err <= 5e-2 * max(1.0, np.abs(st_ref.last_logits).max()), last_err
    assert decidable.mean() >= 0.5, decidable.mean()  # the decision check is not vacuous
