"""CPU-only checks of the product's host layer and C ABI (no GPU needed):
the shared library loads and exports every symbol include/propd.h declares,
tree templates / planning match the oracle, and the multi-rank engine control
flow (gloo, world size 2) reproduces the single-process reference exactly."""

import json
import math
import os
import random
import re

import numpy as np
import pytest
import torch

from oracle import treedecode_port as op
from paper_2402_13485_b200 import _lib
from paper_2402_13485_b200.config import EngineConfig, PruneConfig, SchedulerConfig
from paper_2402_13485_b200.planning import (CostModel, HeadPredictions, InsufficientDataError, choose_size,
                                            grid_candidates, prewarm_P)
from paper_2402_13485_b200.tree import TreeTemplate, canonical_order, mask_to_bits

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ------------------------------------------------------------------ C ABI
def header_functions():
    text = open(os.path.join(ROOT, "include", "propd.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    out = {}
    for m in re.finditer(r"(?:int64_t|int|const char\*)\s+(propd_\w+)\s*\(([^)]*)\)\s*;", text):
        args = [a for a in m.group(2).split(",") if a.strip() and a.strip() != "void"]
        out[m.group(1)] = len(args)
    return out


def test_library_exports_every_header_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libpropd.so not built (run __graft_entry__.build())")
    lib = _lib.load()
    decl = header_functions()
    assert len(decl) >= 20
    for name, nargs in decl.items():
        assert hasattr(lib, name), name
        if name in _lib.SIGNATURES:
            assert len(_lib.SIGNATURES[name]) == nargs, (name, nargs, len(_lib.SIGNATURES[name]))
    assert set(_lib.SIGNATURES) <= set(decl)
    assert lib.propd_abi_version() == _lib.ABI_VERSION


def test_load_fails_loudly_without_library(monkeypatch, tmp_path):
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(ImportError, match="no CPU fallback"):
        _lib.load()


# ------------------------------------------------------------------ trees
def test_templates_match_oracle_build_tree():
    rng = np.random.default_rng(0)
    for _ in range(200):
        D, k = int(rng.integers(1, 5)), int(rng.integers(1, 5))
        sel = op.complete_tree_paths(D, k)
        keep = set()
        for p in sorted(sel, key=len):
            if (len(p) == 1 or p[:-1] in keep) and rng.random() < 0.5:
                keep.add(p)
        if not keep:
            keep = {(1,)}
        preds = op.Preds(np.arange(D * k).reshape(D, k) + 10, -np.tile(np.arange(float(k)), (D, 1)))
        tree = op.build_tree(preds, keep, root_token=0)
        t = TreeTemplate.from_paths(keep, D, k)
        assert list(t.parent) == tree.parents.tolist()
        assert list(t.depth) == tree.depths.tolist()
        assert [n.rank for n in tree.nodes] == list(t.rank)
        assert np.array_equal(t.mask(), op.make_mask(tree))
        assert np.array_equal(mask_to_bits(op.make_mask(tree)), t.mask_bits)
        parents_with_kids = sorted({n.parent for n in tree.nodes if n.parent >= 0})
        assert list(t.parent_nodes) == parents_with_kids


def test_canonical_order_rejects_open_selection():
    with pytest.raises(ValueError, match="ancestor-closed"):
        canonical_order([(1,), (2, 1)])


def test_format_mask_golden(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "gate_numbers.json")))
    t = TreeTemplate.from_paths({(1,), (1, 1), (1, 2), (1, 1, 1)})
    assert op.format_mask(t.mask()) == g["fig_mask"]


# ------------------------------------------------------------------ planning
def test_grid_and_prewarm_match_oracle():
    for D, k in [(1, 1), (4, 3), (3, 16), (4, 64)]:
        assert grid_candidates(D, k) == op.grid_candidates(D, k)
        assert np.array_equal(prewarm_P(D, k), op.Stats(D, k).P)


def test_cost_model_and_choose_size_match_oracle():
    rng = random.Random(7)
    for _ in range(300):
        sizes = sorted(rng.sample(range(1, 65), rng.randint(2, 8)))
        a, lam = rng.choice([0.2, 1.0]), rng.choice([0.0, 0.01])
        mine, ref = CostModel(sizes, alpha=a, staleness_decay=lam), op.Cost(sizes, alpha=a, staleness_decay=lam)
        for now in range(1, rng.randint(2, 30)):
            s = rng.choice(sizes)
            t = rng.uniform(1, 5)
            mine.observe(s, t, now)
            ref.observe(s, t, now)
        now += 1
        try:
            b_ref = ref.fit(now)
        except op.NoFit:
            with pytest.raises(InsufficientDataError):
                mine.fit(now)
            continue
        assert mine.fit(now) == b_ref
        curve = {s: v for s, v in zip(sizes, np.cumsum([rng.uniform(0.05, 1) for _ in sizes]))}
        inc = rng.random() < 0.5
        assert choose_size(curve, mine, inc) == op.choose_size(curve, ref, inc)


def test_head_predictions_validation_messages():
    with pytest.raises(ValueError, match="duplicate"):
        HeadPredictions([[1, 1]], [[0.0, -1.0]])
    with pytest.raises(ValueError, match="non-increasing"):
        HeadPredictions([[1, 2]], [[0.0, 1.0]])
    p = HeadPredictions([[9, 4, 7]], [[0.5, 0.3, 0.2]])
    assert p.rank_of(1, 4) == 2 and p.rank_of(1, 123) is None and p.token(1, 3) == 7


def test_engine_config_validation_matches_reference():
    with pytest.raises(ValueError, match="unknown mode"):
        EngineConfig(mode="nope")
    with pytest.raises(ValueError, match="needs a prune config"):
        EngineConfig(mode="propd_full")
    with pytest.raises(ValueError):
        PruneConfig(layer=0)
    with pytest.raises(ValueError):
        SchedulerConfig(size_candidates=())


def test_neumaier_prefix_sums_equal_cpython_sum():
    """The device l-curve (propd_stats_replay_select) restates CPython's
    compensated float sum(); check the restatement on adversarial inputs."""
    rng = random.Random(3)
    for _ in range(5000):
        xs = [rng.random() ** rng.randint(1, 8) * rng.choice([1, 1e-8, 1e8]) for _ in range(rng.randint(1, 48))]
        f, c, out = xs[0], 0.0, [xs[0]]
        for x in xs[1:]:
            t = f + x
            c += ((f - t) + x) if abs(f) >= abs(x) else ((x - t) + f)
            f = t
            out.append(f + c if (c != 0.0 and math.isfinite(c)) else f)
        assert out == [sum(xs[:s]) for s in range(1, len(xs) + 1)]


# ------------------------------------------------------------------ multi-rank (gloo)
def _gloo_worker(rank, world, port, mode, result_path):
    import torch.distributed as dist

    from paper_2402_13485_b200.engine import DecodeEngine
    from tests.fake_backend import OracleBatchBackend

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2402_13485_b200 import parallel

        # the one per-step collective: fixed-size tables, rows in rank (= global sequence) order
        rows = np.full((rank + 1, parallel.record_width(2)), rank + 1, dtype=np.int32)
        table = parallel.step_exchange(rows, 100 * (rank + 1), 2, dist.group.WORLD)
        assert tuple(table.shape) == (2, 3, parallel.record_width(2))
        hrows, step_us, _ = parallel.global_rows(table)
        assert hrows.shape[0] == 3 and (hrows[:1] == 1).all() and (hrows[1:] == 2).all()
        assert step_us.tolist() == [100, 200]
        cfg = op.RUN_TINY
        e = cfg["engine"]
        ecfg = EngineConfig(mode=mode, draft_heads=4, draft_topk=3,
                            prune=PruneConfig(e.prune.layer, e.prune.topk) if mode in ("prune_only", "propd_full")
                            else None,
                            scheduler=SchedulerConfig(replan_period=16, size_candidates=(1, 2, 4, 6, 8, 10, 12)))
        eng = DecodeEngine(OracleBatchBackend(cfg["model"]), ecfg, op.Clock(**cfg["clock"]), group=dist.group.WORLD)
        w = cfg["workload"]
        prompts = op.synthetic_prompts(256, w["num_prompts"], w["prompt_len"], w["seed"])
        res = eng.run(prompts, w["max_tokens"], batch_size=w["batch_size"])
        if rank == 0:
            with open(result_path, "w") as fh:
                json.dump({"transcripts": res.transcripts, "metrics": [m.to_json() for m in res.metrics],
                           "P": eng.stats_P.tolist() if ecfg.uses_tree else None}, fh)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["propd_full", "static_tree", "autoregressive"])
def test_two_rank_sharded_engine_equals_single_process_reference(golden_dir, tmp_path, mode):
    import torch.multiprocessing as mp

    port = 29500 + random.Random(mode).randint(0, 2000)
    out = tmp_path / "rank0.json"
    mp.spawn(_gloo_worker, args=(2, port, mode, str(out)), nprocs=2, join=True)
    got = json.load(open(out))
    g = json.load(open(os.path.join(golden_dir, f"run_tiny_{mode}.json")))
    assert got["transcripts"] == g["transcripts"]
    assert [json.dumps(m) for m in got["metrics"]] == [json.dumps(m) for m in g["metrics"]]
    if got["P"] is not None:
        assert np.array_equal(np.array(got["P"]), np.array(g["final_P"]))
