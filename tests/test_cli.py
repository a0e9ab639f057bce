"""The reference-format front end (paper_2402_13485_b200.cli): config loading,
the seeded latency clock, and the output files — byte-identical to the real
reference CLI's outputs for configs/run_tiny.json (tests/golden/cli_*, made by
oracle/make_golden.py from the unmodified reference)."""

import json
import os
from types import SimpleNamespace

import pytest

from oracle import treedecode_port as op
from paper_2402_13485_b200 import cli
from paper_2402_13485_b200.planning import LatencyModel

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
RUN_FILES = ["metrics.jsonl", "summary.csv", "plan_events.jsonl"] + [f"transcript_{i:03d}.txt" for i in range(8)]


def _read(path):
    with open(path) as fh:
        return fh.read()


def test_config_and_prompts_match_reference_builders():
    cfg = cli.load_config(os.path.join(GOLD, "run_tiny_config.json"))
    ecfg = cli.build_engine_config(cfg)
    assert ecfg.mode == "propd_full" and ecfg.prune.layer == 2 and ecfg.prune.topk == 24
    assert ecfg.scheduler.size_candidates == (1, 2, 4, 6, 8, 10, 12) and ecfg.draft_topk == 3
    gold = json.load(open(os.path.join(GOLD, "run_tiny_propd_full.json")))
    assert cli.build_prompts(cfg, 256) == gold["prompts"]


def test_latency_model_matches_oracle_clock():
    a = LatencyModel(c0_base=3.0, c1_base=0.05, noise=0.02, c0_batch=0.1, seed=4)
    b = op.Clock(c0_base=3.0, c1_base=0.05, noise=0.02, c0_batch=0.1, seed=4)
    for i in range(50):
        assert a.iteration_time(i * 0.7, batch=1 + i % 5, seqlen=30.0 + i) == b.iteration_time(
            i * 0.7, batch=1 + i % 5, seqlen=30.0 + i)
    with pytest.raises(ValueError, match="non-negative"):
        LatencyModel(noise=-1)


def test_output_writer_is_byte_identical(tmp_path):
    """The writer fed with the reference's own run record reproduces the reference CLI's files."""
    gold = json.load(open(os.path.join(GOLD, "run_tiny_propd_full.json")))
    metrics = [SimpleNamespace(to_json=(lambda m=m: m)) for m in gold["metrics"]]
    events = [SimpleNamespace(iteration=e["iteration"], trigger=e["trigger"], chosen_size=e["chosen_size"],
                              l_curve=e["l_curve"], v_curve=e["v_curve"]) for e in gold["plan_events"]]
    result = SimpleNamespace(prompts=gold["prompts"], transcripts=gold["transcripts"], metrics=metrics,
                             plan_events=events, summary=SimpleNamespace(**gold["summary"]))
    cfg = cli.load_config(os.path.join(GOLD, "run_tiny_config.json"))
    cli.write_outputs(tmp_path, cfg, result, verbose=True)
    for f in RUN_FILES:
        assert _read(tmp_path / f) == _read(os.path.join(GOLD, "cli_run_tiny", f)), f


def test_config_errors_exit_2(tmp_path, capsys):
    bad = tmp_path / "bad.json"
    bad.write_text('{"backend": {"kind": "synthetic"}}')
    assert cli.main(["run", "--config", str(bad)]) == 2
    assert "not served by the B200 backend" in capsys.readouterr().err
    bad.write_text('{"engine": {"mode": "fastest"}}')
    assert cli.main(["run", "--config", str(bad)]) == 2
    bad.write_text("{\n  oops")
    assert cli.main(["run", "--config", str(bad)]) == 2
    assert ":2: invalid JSON" in capsys.readouterr().err


@pytest.mark.gpu
def test_cli_run_and_sweep_on_b200_match_reference_files(tmp_path):
    """`run` on the B200 backend (fp32 parity mode) writes the reference CLI's files byte for byte;
    `sweep` reproduces its sweep.csv (simulated clock, in-process AR baseline)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    out = tmp_path / "run"
    assert cli.main(["run", "--config", os.path.join(GOLD, "run_tiny_config.json"), "--out-dir", str(out),
                     "--verbose"]) == 0
    for f in RUN_FILES:
        assert _read(out / f) == _read(os.path.join(GOLD, "cli_run_tiny", f)), f
    sw = tmp_path / "sweep"
    assert cli.main(["sweep", "--config", os.path.join(GOLD, "sweep_tiny_config.json"), "--axis", "mode",
                     "--axis", "batch", "--out-dir", str(sw)]) == 0
    assert _read(sw / "sweep.csv") == _read(os.path.join(GOLD, "cli_sweep_tiny", "sweep.csv"))
