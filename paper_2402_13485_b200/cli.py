"""Command-line front end with the reference's config format and output files,
running the decode loop on the B200 backend.

Mirrors `treedecode.cli` (paths relative to /root/reference/pkg/src/treedecode/):
  run    cli.py:86-98   -> transcript_NNN.txt, metrics.jsonl, summary.csv
                          (+ plan_events.jsonl with --verbose), cli.py:27-73
  sweep  cli.py:118-171 -> sweep.csv with the in-process autoregressive
                          baseline and a speedup column
Config: the reference JSON layout and defaults (config.py:173-207, 266-354).
`backend.kind` "tiny" builds the reference's seeded TinyTransformer weights
(fp32 parity mode by default); "b200" builds a model of any shape
(`backend.b200`: layers, hidden, heads, vocab, draft_heads, max_positions,
dtype, random_init, planted_draft_head) — e.g. the Vicuna-7B shape in bf16.
The SyntheticOracle backend is a CPU test fixture of the reference and is not
offered here.

  python -m paper_2402_13485_b200.cli run --config run.json [--out-dir D]
  python -m paper_2402_13485_b200.cli sweep --config s.json --axis batch [--axis mode]
"""

from __future__ import annotations

import argparse
import copy
import csv
import itertools
import json
import sys
from pathlib import Path

import numpy as np

from .config import EngineConfig, PruneConfig, SchedulerConfig, TinyTransformerConfig
from .planning import LatencyModel


class ConfigError(ValueError):
    """A configuration problem; reported as `config error: ...`, exit status 2."""


DEFAULTS = {
    "backend": {"kind": "tiny", "seed": 0, "tiny": {}, "b200": {}, "latency": {}},
    "engine": {"mode": "propd_full", "draft_heads": 4, "draft_topk": 3, "prune": None, "scheduler": {},
               "static_tree": None, "acceptance_alpha": 0.05, "cost_alpha": 0.2, "cost_staleness": 0.01,
               "include_bonus_in_speed": False, "probe_rounds": 1, "eos_token": None, "clock": "model"},
    "workload": {"kind": "synthetic", "num_prompts": 16, "prompt_len": 8, "path": None, "max_tokens": 32,
                 "batch_size": None, "seed": 1},
    "output": {"dir": "out", "transcripts": True, "metrics": True, "summary": True},
    "sweep": {},
}
AXES = ("batch", "mode", "prune_layer", "prune_topk")


def load_config(path) -> dict:
    """JSON config merged over the reference defaults (section by section)."""
    path = Path(path)
    try:
        raw = json.loads(path.read_text())
    except OSError as exc:
        raise ConfigError(f"{path}: {exc}") from exc
    except json.JSONDecodeError as exc:
        raise ConfigError(f"{path}:{exc.lineno}: invalid JSON: {exc.msg}") from exc
    if not isinstance(raw, dict):
        raise ConfigError(f"{path}: top level must be an object")
    cfg = copy.deepcopy(DEFAULTS)
    for section, body in raw.items():
        if section not in cfg:
            raise ConfigError(f"{path}: {section}: unknown section")
        if isinstance(cfg[section], dict) and isinstance(body, dict):
            cfg[section].update(body)
        else:
            raise ConfigError(f"{path}: {section}: must be an object")
    if cfg["backend"]["kind"] not in ("tiny", "b200"):
        raise ConfigError(f"backend.kind: {cfg['backend']['kind']!r} is not served by the B200 backend "
                          "(expected 'tiny' or 'b200')")
    return cfg


def apply_seed_override(cfg: dict, seed) -> dict:
    """Re-seed backend, latency model and workload (config.py:255-263)."""
    if seed is None:
        return cfg
    out = copy.deepcopy(cfg)
    out["backend"]["seed"] = seed
    out["backend"]["latency"].pop("seed", None)
    out["workload"]["seed"] = seed
    return out


def build_backend(cfg: dict, max_slots: int):
    from .backend import B200Backend

    section = cfg["backend"]
    seed = section["seed"]
    try:
        if section["kind"] == "tiny":
            mcfg = TinyTransformerConfig(seed=seed, **section["tiny"])
            return B200Backend(mcfg, dtype="fp32", max_slots=max_slots)
        params = dict(section["b200"])
        dtype = params.pop("dtype", "bf16")
        random_init = bool(params.pop("random_init", True))
        planted = params.pop("planted_draft_head", False)
        mcfg = TinyTransformerConfig(seed=seed, **params)
        be = B200Backend(mcfg, dtype=dtype, random_device_init=random_init, max_slots=max_slots,
                         use_graphs=dtype == "bf16")
        if planted:
            be.plant_draft_head(0)
        return be
    except (TypeError, ValueError) as exc:
        raise ConfigError(f"backend.{section['kind']}: {exc}") from exc


def build_latency(cfg: dict):
    """The engine clock: the seeded latency model, or None for wall time."""
    if cfg["engine"]["clock"] == "wall":
        return None
    params = dict(cfg["backend"]["latency"])
    params.setdefault("seed", cfg["backend"]["seed"] + 1)
    try:
        return LatencyModel(**params)
    except (TypeError, ValueError) as exc:
        raise ConfigError(f"backend.latency: {exc}") from exc


def build_engine_config(cfg: dict) -> EngineConfig:
    s = cfg["engine"]
    try:
        prune = PruneConfig(**s["prune"]) if s["prune"] else None
        sched = SchedulerConfig(**{k: tuple(v) if k == "size_candidates" else v for k, v in s["scheduler"].items()})
        static = tuple(tuple(p) for p in s["static_tree"]) if s["static_tree"] else None
        return EngineConfig(mode=s["mode"], draft_heads=s["draft_heads"], draft_topk=s["draft_topk"], prune=prune,
                            scheduler=sched, static_tree=static, acceptance_alpha=s["acceptance_alpha"],
                            cost_alpha=s["cost_alpha"], cost_staleness=s["cost_staleness"],
                            include_bonus_in_speed=s["include_bonus_in_speed"], probe_rounds=s["probe_rounds"],
                            eos_token=s["eos_token"], acceptance=s.get("acceptance", "greedy"),
                            typical_epsilon=s.get("typical_epsilon", 0.09), typical_alpha=s.get("typical_alpha", 0.3),
                            typical_temperature=s.get("typical_temperature", 1.0))
    except (TypeError, ValueError) as exc:
        raise ConfigError(f"engine: {exc}") from exc


def build_prompts(cfg: dict, vocab: int) -> list:
    s = cfg["workload"]
    if s["kind"] == "file":
        if not s["path"]:
            raise ConfigError("workload.path: required when workload.kind is 'file'")
        try:
            data = json.loads(Path(s["path"]).read_text())
        except (OSError, json.JSONDecodeError) as exc:
            raise ConfigError(f"workload.path: {exc}") from exc
        if not (isinstance(data, list) and data and all(
                isinstance(p, list) and p and all(isinstance(t, int) and 0 <= t < vocab for t in p) for p in data)):
            raise ConfigError(f"{s['path']}: prompt file must be a non-empty JSON array of non-empty arrays of "
                              f"token ids below {vocab}")
        return [list(p) for p in data]
    rng = np.random.default_rng(s["seed"])
    return [rng.integers(0, vocab, size=s["prompt_len"]).tolist() for _ in range(s["num_prompts"])]


def run_once(cfg: dict):
    from .engine import DecodeEngine

    w = cfg["workload"]
    b = cfg["backend"]
    vocab = (b["tiny"] if b["kind"] == "tiny" else b["b200"]).get("vocab", TinyTransformerConfig().vocab)
    ecfg, latency = build_engine_config(cfg), build_latency(cfg)  # validate before touching the device
    prompts = build_prompts(cfg, vocab)
    # the engine holds one batch chunk at a time and frees its slots after it
    # (the backend adds its own scratch slot for padded rows)
    bs = w["batch_size"]
    backend = build_backend(cfg, max_slots=len(prompts) if bs is None else min(max(1, int(bs)), len(prompts)))
    engine = DecodeEngine(backend, ecfg, latency)
    result = engine.run(prompts, w["max_tokens"], batch_size=w["batch_size"])
    return engine, result


def write_outputs(out_dir: Path, cfg: dict, result, verbose: bool) -> None:
    """The reference's run outputs, byte for byte in format (cli.py:27-73)."""
    out_dir.mkdir(parents=True, exist_ok=True)
    out = cfg["output"]
    if out["transcripts"]:
        for i, (prompt, gen) in enumerate(zip(result.prompts, result.transcripts)):
            (out_dir / f"transcript_{i:03d}.txt").write_text(
                " ".join(str(t) for t in prompt) + "\n" + " ".join(str(t) for t in gen) + "\n")
    if out["metrics"]:
        with (out_dir / "metrics.jsonl").open("w") as fh:
            for m in result.metrics:
                fh.write(json.dumps(m.to_json()) + "\n")
    if out["summary"]:
        s = result.summary
        with (out_dir / "summary.csv").open("w", newline="") as fh:
            wr = csv.writer(fh)
            wr.writerow(["mode", "iterations", "total_tokens", "total_time", "tokens_per_sec", "mean_accepted",
                         "mean_prune_rate", "mean_tree_size"])
            wr.writerow([s.mode, s.iterations, s.total_tokens, f"{s.total_time:.6f}", f"{s.tokens_per_sec:.6f}",
                         f"{s.mean_accepted:.6f}", f"{s.mean_prune_rate:.6f}", f"{s.mean_tree_size:.6f}"])
    if verbose:
        with (out_dir / "plan_events.jsonl").open("w") as fh:
            for ev in result.plan_events:
                fh.write(json.dumps({"iteration": ev.iteration, "trigger": ev.trigger, "chosen_size": ev.chosen_size,
                                     "l_curve": {str(k): v for k, v in ev.l_curve.items()},
                                     "v_curve": {str(k): v for k, v in ev.v_curve.items()}}) + "\n")


def cmd_run(args) -> int:
    cfg = apply_seed_override(load_config(args.config), args.seed_override)
    _, result = run_once(cfg)
    out_dir = Path(args.out_dir or cfg["output"]["dir"])
    write_outputs(out_dir, cfg, result, args.verbose)
    s = result.summary
    print(f"mode={s.mode} iterations={s.iterations} tokens={s.total_tokens} time={s.total_time:.3f} "
          f"tokens_per_sec={s.tokens_per_sec:.3f} mean_accepted={s.mean_accepted:.3f}")
    print(f"outputs written to {out_dir}")
    return 0


def _apply_axis(cfg: dict, axis: str, value) -> dict:
    out = copy.deepcopy(cfg)
    if axis == "batch":
        out["workload"]["batch_size"] = value
    elif axis == "mode":
        out["engine"]["mode"] = value
    else:
        if not out["engine"]["prune"]:
            raise ConfigError(f"sweep.{axis}: engine.prune must be configured for this axis")
        out["engine"]["prune"]["layer" if axis == "prune_layer" else "topk"] = value
    return out


def cmd_sweep(args) -> int:
    cfg = apply_seed_override(load_config(args.config), args.seed_override)
    axes = list(dict.fromkeys(args.axis))
    for axis in axes:
        if not cfg["sweep"].get(axis):
            raise ConfigError(f"sweep.{axis}: no values configured for this axis")
    rows = []
    for combo in itertools.product(*[cfg["sweep"][a] for a in axes]):
        run_cfg = cfg
        for axis, value in zip(axes, combo):
            run_cfg = _apply_axis(run_cfg, axis, value)
        _, result = run_once(run_cfg)
        base_cfg = copy.deepcopy(run_cfg)
        base_cfg["engine"]["mode"] = "autoregressive"
        _, baseline = run_once(base_cfg)
        s = result.summary
        row = dict(zip(axes, combo))
        row.update({"mode": s.mode, "total_tokens": s.total_tokens, "total_time": s.total_time,
                    "tokens_per_sec": s.tokens_per_sec, "mean_accepted": s.mean_accepted,
                    "mean_prune_rate": s.mean_prune_rate, "baseline_time": baseline.summary.total_time,
                    "speedup": baseline.summary.total_time / s.total_time if s.total_time > 0 else float("nan")})
        rows.append(row)
    print(f"sweep axes: {', '.join(axes)}")
    for r in rows:
        cells = " ".join(f"{r[a]!s:>12}" for a in axes)
        print(f"{cells} {r['mode']:>14} {r['total_tokens']:>8} {r['total_time']:>10.3f} {r['tokens_per_sec']:>10.3f} "
              f"{r['mean_accepted']:>8.3f} {r['mean_prune_rate']:>7.3f} {r['speedup']:>8.3f}")
    out_dir = Path(args.out_dir or cfg["output"]["dir"])
    out_dir.mkdir(parents=True, exist_ok=True)
    with (out_dir / "sweep.csv").open("w", newline="") as fh:
        wr = csv.DictWriter(fh, fieldnames=list(rows[0].keys()))
        wr.writeheader()
        for r in rows:
            wr.writerow({k: (f"{v:.6f}" if isinstance(v, float) else v) for k, v in r.items()})
    print(f"wrote {out_dir / 'sweep.csv'}")
    return 0


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="paper_2402_13485_b200",
                                description="ProPD tree decoding on B200 (reference config and output formats).")
    sub = p.add_subparsers(dest="command", required=True)
    run = sub.add_parser("run", help="decode a workload under one engine mode")
    run.add_argument("--config", required=True)
    run.add_argument("--out-dir", default=None)
    run.add_argument("--seed-override", type=int, default=None)
    run.add_argument("--verbose", action="store_true", help="also write plan_events.jsonl")
    run.set_defaults(func=cmd_run)
    sw = sub.add_parser("sweep", help="run config axes across their configured values")
    sw.add_argument("--config", required=True)
    sw.add_argument("--axis", required=True, action="append", choices=AXES)
    sw.add_argument("--out-dir", default=None)
    sw.add_argument("--seed-override", type=int, default=None)
    sw.set_defaults(func=cmd_sweep)
    return p


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except ConfigError as exc:
        print(f"config error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
