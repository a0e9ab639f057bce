"""Two ranks, one B200Backend each, sharing one GPU over a gloo process group
(the box has one GPU; NCCL between two processes on one device is not
supported): the sequence-sharded decode loop with its single per-step
all-gather (paper_2402_13485_b200/parallel.py) must reproduce the
single-process reference exactly — transcripts, per-iteration metrics and the
fp64 acceptance statistics P (engine.py:257-303, acceptance.py:96-113) — from
the real reference's goldens (tests/golden, oracle/make_golden.py)."""

import json
import os
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import treedecode_port as op  # noqa: E402


def _worker(rank, world, port, mode, result_path):
    import torch.distributed as dist

    from paper_2402_13485_b200 import (B200Backend, DecodeEngine, EngineConfig, PruneConfig, SchedulerConfig,
                                       TinyTransformerConfig)

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        cfg = op.RUN_TINY
        e = cfg["engine"]
        ecfg = EngineConfig(mode=mode, draft_heads=4, draft_topk=3,
                            prune=PruneConfig(e.prune.layer, e.prune.topk) if mode in ("prune_only", "propd_full")
                            else None,
                            scheduler=SchedulerConfig(replan_period=16, size_candidates=(1, 2, 4, 6, 8, 10, 12)))
        be = B200Backend(TinyTransformerConfig(**cfg["model"].__dict__), dtype="fp32", device="cuda:0", max_slots=8,
                         use_graphs=True)
        eng = DecodeEngine(be, ecfg, op.Clock(**cfg["clock"]), group=dist.group.WORLD)
        w = cfg["workload"]
        prompts = op.synthetic_prompts(256, w["num_prompts"], w["prompt_len"], w["seed"])
        res = eng.run(prompts, w["max_tokens"], batch_size=w["batch_size"])
        with open(f"{result_path}.{rank}", "w") as fh:
            json.dump({"transcripts": res.transcripts, "metrics": [m.to_json() for m in res.metrics],
                       "P": eng.stats_P.tolist() if ecfg.uses_tree else None,
                       "native": be.launches}, fh)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["propd_full", "static_tree"])
def test_two_rank_b200_engine_equals_single_process_reference(golden_dir, tmp_path, mode):
    import torch.multiprocessing as mp

    port = 31000 + random.Random(mode).randint(0, 2000)
    out = str(tmp_path / "rank")
    mp.spawn(_worker, args=(2, port, mode, out), nprocs=2, join=True)
    g = json.load(open(os.path.join(golden_dir, f"run_tiny_{mode}.json")))
    for r in range(2):
        got = json.load(open(f"{out}.{r}"))
        assert got["native"] > 0  # the kernels ran on both ranks
        assert got["transcripts"] == g["transcripts"]  # every rank holds every transcript
        assert [json.dumps(m) for m in got["metrics"]] == [json.dumps(m) for m in g["metrics"]]
        assert np.array_equal(np.array(got["P"]), np.array(g["final_P"]))
