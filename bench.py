"""Benchmark of the batched ProPD decode step on B200 (contract: one JSON line).

Workload (BASELINE.json configs[1]): Vicuna-7B-shape random-init bf16 model
(32 layers, hidden 4096, 32 heads x 128, vocab 32000, 4 draft heads),
batch 1 per GPU, synthetic prompt state of KV length --kv (default 1024),
ProPD pruned + dynamic tree (propd_full: prune layer 4, top-K 50, k=16
candidates per head -> grid of 64 nodes).  A step = one engine iteration
(draft, plan, tree pass with early pruning, greedy accept + KV compaction,
bonus pass, on-device statistics replay) over the whole batch.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

N>1: bench.py re-launches itself under torchrun (one rank per GPU, NCCL),
sequences sharded (weak scaling: --batch is per GPU), one all-gather of the
per-step record table per step.  `value` = committed tokens of all ranks /
max-over-ranks device time.  At N=1 the line also carries `sweep`: the
north-star grid (configs[2]: B 1-64 x KV 1024/4096, static Medusa tree vs
ProPD at B=1) measured in the same process.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode tokens/sec @ batch 1-64 (7B shape); accepted len/step; verify ms/step"
SIZES = (1, 2, 4, 8, 16, 32, 64)


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--batch", type=int, default=1, help="sequences per GPU")
    ap.add_argument("--kv", type=int, default=1024, help="KV length (synthetic prompt state)")
    ap.add_argument("--mode", default="propd_full")
    ap.add_argument("--topk", type=int, default=16, help="draft top-k per head (tree grid = 4 x topk)")
    ap.add_argument("--shape", default="7b", choices=["7b", "33b"],
                    help="Vicuna-7B shape (configs[1-2]) or Vicuna-33B shape (configs[3]: 60 x 6656, 52 heads)")
    ap.add_argument("--layers", type=int, default=None, help="override the shape's layer count")
    ap.add_argument("--attn-impl", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the north-star grid (N=1 only)")
    ap.add_argument("--sweep-points", default="1:1024:propd_full,1:1024:static_tree,1:4096,8:1024,8:4096,32:1024,"
                                               "32:4096,64:4096",
                    help="B:KV[:mode] points of the in-process sweep")
    ap.add_argument("--no-graphs", action="store_true", help="eager launches instead of CUDA graphs")
    ap.add_argument("--acceptance", default="greedy", choices=["greedy", "typical"])
    ap.add_argument("--prune-threshold", type=float, default=None,
                    help="probability-based pruning (marginal path probability >= threshold) instead of top-K 50")
    ap.add_argument("--planted", action="store_true",
                    help="planted acceptance (SURVEY f3): draft head 0 := LM head, so depth-1 nodes are accepted")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend under torchrun (gloo + --same-device: a multi-rank dry run on 1 GPU)")
    ap.add_argument("--same-device", action="store_true", help="every rank on cuda:0 (multi-rank dry run)")
    ap.add_argument("--sync-rows", action="store_true",
                    help="size the post-prune layers on the host (one mid-step sync) instead of on the device")
    ap.add_argument("--ref-tree-sizes", default="64,64,64,64,32,32,32,32,32,32,32,32,32,32,32,32,32,32,32,32",
                    help="reference arm: per-step tree sizes (cycled) it is pinned to; the default is the schedule "
                         "the B200 arm's dynamic plan ran in its 20 timed steps at configs[1] (mean 38.4 nodes)")
    return ap.parse_args(argv)


def model_cfg(args, kv_cap: int | None = None):
    from paper_2402_13485_b200 import VICUNA_7B_SHAPE, VICUNA_33B_SHAPE, TinyTransformerConfig

    shape = dict(VICUNA_7B_SHAPE if getattr(args, "shape", "7b") == "7b" else VICUNA_33B_SHAPE)
    if getattr(args, "layers", None) is not None:
        shape["layers"] = args.layers
    kv = args.kv if kv_cap is None else kv_cap
    # growth room: every step commits acc + 1 tokens (random init: acc ~ 0; planted: 1) over at most four
    # priming phases of <= 48 steps, the warm-up and three K-step regions
    per_step = 3 if getattr(args, "planted", False) else 2
    return TinyTransformerConfig(**shape, max_positions=kv + per_step * (4 * 48 + 3 * args.steps + args.warmup + 8)
                                 + 64, seed=0)


def engine_cfg(args, mode=None):
    from paper_2402_13485_b200 import EngineConfig, PruneConfig, SchedulerConfig

    mode = mode or args.mode
    threshold = getattr(args, "prune_threshold", None)
    prune = PruneConfig(layer=4, topk=50, threshold=threshold) if mode in ("prune_only", "propd_full") else None
    sizes = tuple(s for s in SIZES if s <= 4 * args.topk)
    return EngineConfig(mode=mode, draft_heads=4, draft_topk=args.topk, prune=prune,
                        scheduler=SchedulerConfig(replan_period=16, size_candidates=sizes),
                        acceptance=getattr(args, "acceptance", "greedy"))


class ClockSampler:
    """SM clock + throttle reasons sampled through NVML (in-process, no fork)
    every 100 ms during the timed region."""

    def __init__(self, index: int) -> None:
        self.index, self.samples, self._stop = index, [], threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        except Exception as exc:  # pragma: no cover
            self.samples.append(("error", str(exc)))
            return
        bits = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                "sw_power_cap": 0x4}
        while True:
            try:
                mhz = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((mhz, max_mhz, [k for k, b in bits.items() if r & b]))
            except Exception:
                pass
            if self._stop.wait(0.1):
                break

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        good = [s for s in self.samples if s and s[0] != "error"]
        if not good:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(float(s[0]) for s in good), "sm_max_mhz": float(good[0][1]),
                "reasons": sorted({r for s in good for r in s[2]}), "samples": len(good)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def tensor_peak():
    """Dense bf16 TFLOP/s for kernels timed inside a long step (sustained), and the burst figure."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return (float(p["bf16_tflops_sustained"]), float(p["bf16_tflops"]),
                "measured sustained (MEASURED_PEAKS.json bf16_tflops_sustained; burst beside it)")
    except Exception:
        return 1800.0, 1800.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kind: str, args) -> dict:
    """DRAM bytes of one launch of the dominant kernel from a committed ncu
    capture (dram__bytes_read/write) of this bench configuration
    (profiles/ncu_traffic.json), if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            table = json.load(fh)
    except Exception:
        return {}
    key = f"{kind}:b{args.batch}:kv{args.kv}:{args.mode}" + ("" if args.shape == "7b" else f":{args.shape}")
    return table.get(key, {})


# ---------------------------------------------------------------- CPU reference arm
def cpu_reference(args, steps: int, warmup: int, sizes=None):
    """The reference algorithm on the host cores, on the B200 arm's workload:
    oracle/treedecode_port (the fp64 numpy restatement of treedecode's
    DecodeEngine._step, pinned to the real reference by tests/golden) at the
    model's full width (hidden, heads, vocab), batch --batch, KV --kv, the same
    mode, pruning (layer 4, top-K 50) and draft grid, with the tree size of
    every step pinned to `sizes` (the B200 arm's schedule; the dynamic plan's
    path selection from the running statistics is kept).  Five layers run (4
    before the prune point, 1 after; one layer's weights shared by all five:
    values do not change the work) and every block call is timed, so each
    step is extrapolated to the full depth from MEASURED per-layer times:
    T = T_step - T_blocks + p * t_pre + (L - p) * t_post + L * t_commit."""
    import numpy as np

    # all host threads: torchrun exports OMP_NUM_THREADS=1 to every rank
    cores = os.cpu_count()
    os.environ["OPENBLAS_NUM_THREADS"] = str(cores)
    os.environ["OMP_NUM_THREADS"] = str(cores)
    from oracle import treedecode_port as op

    try:  # numpy may already be loaded (threads fixed at load): resize its BLAS pool
        from threadpoolctl import threadpool_limits
        threadpool_limits(cores)
    except Exception:
        pass
    full = model_cfg(args)
    Lf = full.layers
    p = 4
    mode = args.mode
    prune = op.PruneCfg(layer=p, topk=50, threshold=args.prune_threshold) if mode in ("prune_only",
                                                                                    "propd_full") else None
    Ly = p + 1
    H, V, D = full.hidden, full.vocab, full.draft_heads
    cfg = op.TinyCfg(layers=Ly, hidden=H, heads=full.heads, vocab=V, draft_heads=D,
                     max_positions=args.kv + (D + 1) * (steps + warmup) + 8, seed=0)
    rng = np.random.default_rng(0)
    s = 1.0 / np.sqrt(H)
    blk = {k: rng.standard_normal(sh) * s for k, sh in (("wq", (H, H)), ("wk", (H, H)), ("wv", (H, H)),
                                                         ("wo", (H, H)), ("w1", (H, 4 * H)))}
    blk["w2"] = rng.standard_normal((4 * H, H)) * (0.5 * s)
    head = rng.standard_normal((H, V)) * s
    # the other [H, V] heads and the embedding: independent column permutations of one draw (the draft and
    # early heads must not coincide with the LM head, or acceptance would be planted)
    perm = lambda: np.ascontiguousarray(head[:, rng.permutation(V)])
    w = {"emb": np.ascontiguousarray(perm().T), "pos": rng.standard_normal((cfg.max_positions, H)) * s,
         "blocks": [blk] * Ly, "w_lm": head, "w_early": perm(), "w_draft": [perm() for _ in range(D)]}
    if args.planted:
        w["w_draft"][0] = head
    log: list = []

    class TimedModel(op.TinyModel):
        def block(self, x, li, kc, vc, vis):
            t0 = time.perf_counter()
            out = super().block(x, li, kc, vc, vis)
            log.append((li, time.perf_counter() - t0))
            return out

    model = TimedModel(cfg, weights=w)
    sizes = list(sizes) if sizes else [4 * args.topk]

    class PinnedEngine(op.Engine):
        def _plan(self, B, seqlen):  # size pinned per step; paths = the statistics' best nodes (acceptance.py:186-206)
            if not self.cfg.uses_dynamic:
                return super()._plan(B, seqlen)
            size = min(sizes[(self.it - 1) % len(sizes)], self.cfg.draft_heads * self.cfg.draft_topk)
            return op.select_best_nodes(self.stats, [size])[size][0], False

    ecfg = op.EngineCfg(mode=mode, draft_heads=D, draft_topk=args.topk, prune=prune,
                        scheduler=op.SchedCfg(size_candidates=tuple(x for x in SIZES if x <= D * args.topk)),
                        acceptance=args.acceptance)
    eng = PinnedEngine(model, ecfg, None)
    prompts = [rng.integers(0, V, size=args.kv).tolist() for _ in range(args.batch)]
    seqs = [{"state": model.prefill(pr), "prompt": pr, "gen": [], "done": False} for pr in prompts]
    per_step, toks, acc, tree = [], 0, 0.0, 0.0
    for i in range(warmup + steps):
        log.clear()
        t0 = time.perf_counter()
        m = eng.step(seqs, 10 ** 9)
        dt = time.perf_counter() - t0
        if i < warmup:
            continue
        # block calls: the tree pass (Ly per sequence, in order) then each commit's extend (Ly)
        t_blocks = sum(t for _, t in log)
        per_seq = [log[j: j + 2 * Ly] for j in range(0, len(log), 2 * Ly)]
        extr = dt - t_blocks
        for calls in per_seq:
            tree_calls, commit_calls = calls[:Ly], calls[Ly:]
            if prune is not None:
                t_pre = sum(t for _, t in tree_calls[:p]) / p
                t_post = sum(t for _, t in tree_calls[p:]) / (Ly - p)
                extr += p * t_pre + (Lf - p) * t_post
            else:
                extr += Lf * sum(t for _, t in tree_calls) / Ly
            extr += Lf * sum(t for _, t in commit_calls) / max(1, len(commit_calls))
        per_step.append(extr)
        toks += m["tokens_committed"]
        acc += m["mean_accepted"]
        tree += m["tree_size"]
    total = sum(per_step)
    sample = (f"oracle/treedecode_port (fp64 numpy restatement of the reference DecodeEngine._step) at "
              f"{args.shape.upper()} width (hidden {H}, {full.heads} heads, vocab {V}), batch {args.batch}, KV {args.kv}, "
              f"{mode}" + (f" (prune layer {p}, top-K 50)" if prune is not None else "") +
              f", tree size pinned per step to {sizes} (the B200 arm's schedule), {steps} steps timed after {warmup} "
              f"warm-up; {Ly} layers run ({p} before the prune point), every block timed, each step extrapolated to "
              f"{Lf} layers from the measured per-layer times; OPENBLAS_NUM_THREADS={cores}")
    return {"value": toks / total, "unit": "tokens/s", "cores": cores, "kind": "port", "sample": sample,
            "ms_per_step": total / steps * 1e3, "accepted_len_per_step": acc / steps, "tree_size_mean": tree / steps,
            "steps": steps}


# ---------------------------------------------------------------- B200 arm
def local_device(args):
    import torch

    return torch.device("cuda", 0 if args.same_device else int(os.environ.get("LOCAL_RANK", 0)))


def all_max(value: float, group, dev) -> float:
    """Max over ranks (identity without a process group)."""
    if group is None:
        return float(value)
    import torch
    import torch.distributed as dist

    where = dev if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=where)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def attn_step_bytes(be, m, prune_layer) -> float:
    """Algorithmic K2 bytes of one engine step from its metrics:
    per layer and sequence 2 (L_b + r_b) H elt of cache + tree K/V read plus
    r_b H elt of Q read and O written; tree pass r = n (layers <= p) / |S_b|
    (layers > p), bonus pass r = 1 over L_b + acc_b + 1 keys."""
    H, Ly = be.H, be.num_layers
    elt = 2 if be.tdtype != be.torch.float32 else 4
    B, n = m.batch, m.tree_size
    L0 = m.mean_seqlen * B
    f = lambda keys, rows, cap: ((2 * keys + 2 * rows) * H * elt +
                                 fold_bytes(be, rows, cap, B, keys / max(1, B)))
    if n == 0:  # autoregressive
        return 0.0 if bonus_fused(be, B) else Ly * f(L0 + B, B, 1)
    p = prune_layer if prune_layer is not None else Ly
    S = m.mean_survivors * B
    tree = p * f(L0 + B * n, B * n, n) + (Ly - p) * f(L0 + B * n, S, n)
    return tree + (0 if bonus_fused(be, B) else bonus_attn_bytes(be, m))


def fold_bytes(be, rows, cap=1, nseq=1, keys=0) -> float:
    """Extra algorithmic bytes of a pass whose QKV tail is folded into the
    attention (B200Backend.ws_qkv_fold: weight-streaming passes of <= 128
    rows; cap = row capacity per sequence): the kernel reads its rows' fp32
    Q / K / V (3 H x 4 B) and writes their bf16 K/V (2 H x 2 B) instead of
    reading a bf16 Q (H x 2 B)."""
    if not (getattr(be, "ws_qkv_fold", False) and be.tdtype != be.torch.float32 and nseq * cap <= 128):
        return 0.0
    return rows * be.H * (12 + 4 - 2)


def bonus_fused(be, B) -> bool:
    """The bonus pass's attention runs inside its QKV launches (one-row fusion)."""
    return bool(getattr(be, "ws_fuse_attn", False)) and be.fused_one_row_splits(B) > 0


def bonus_attn_bytes(be, m) -> float:
    """Algorithmic K/V + q/o bytes of the bonus pass's attention (all layers)."""
    elt = 2 if be.tdtype != be.torch.float32 else 4
    B = m.batch
    keys = m.mean_seqlen * B + m.mean_accepted * B + B
    return be.num_layers * ((2 * keys + 2 * B) * be.H * elt + fold_bytes(be, B, 1, B, keys / max(1, B)))


def modal_size(metrics):
    """Most frequent tree size of the timed steps (None without steps)."""
    sizes = [x.tree_size for x in metrics]
    return max(set(sizes), key=sizes.count) if sizes else None


def timeline_step(be, eng, seqs, prime, dev, prune_layer, tree_size=None):
    """One step with per-CTA globaltimer records (graphs captured with the
    trace on): busy time of each kernel family inside the PDL-chained step =
    union over its launches of [dependency release, last CTA exit]; GEMM bytes
    from the shapes in the trace records (weight stages streamed before a
    launch's release are left out of its window's bytes: conservative),
    attention bytes from the step's metrics.  tree_size: the timed steps'
    (modal) tree size — the dynamic plan may have moved since, so up to 12
    steps are traced until one has that size (`traced_tree_size` reports the
    size of the step actually traced)."""
    import ctypes

    import numpy as np
    import torch

    cap = 1 << 20
    buf = torch.zeros(8 + 8 * cap, device=dev, dtype=torch.int64)
    buf[1] = cap
    lib = be.lib
    lib.propd_debug_timeline(ctypes.c_void_p(buf.data_ptr()))
    be.timeline = buf
    try:
        prime()
        for _ in range(12):
            torch.cuda.synchronize()
            buf[0] = 0
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record()
            m = eng._step(seqs, 10 ** 9)
            t1.record()
            torch.cuda.synchronize()
            if tree_size is None or m.tree_size == tree_size:
                break
    finally:
        lib.propd_debug_timeline(ctypes.c_void_p(0))
        be.timeline = None
    n = min(int(buf[0].item()), cap)
    rec = buf[8: 8 + 8 * n].view(n, 8).cpu().numpy()
    out = {"step_ms": t0.elapsed_time(t1), "records": n, "traced_tree_size": m.tree_size}
    if os.environ.get("PROPD_BENCH_DUMP"):  # development aid: the raw per-CTA records of the traced step
        np.save(os.environ["PROPD_BENCH_DUMP"], rec)
    kinds = rec[:, 7] & 0xFF
    hbm, _ = peaks()
    for kind, name in ((1, "gemm"), (2, "attn"), (5, "gemm_tc")):
        # kind 4 = the transposed attention kernel (same release / exit columns)
        r = rec[(kinds == kind) | ((kinds == 4) if kind == 2 else False)]
        if len(r) == 0:
            continue
        spans = []
        nbytes = flops = 0
        for tag in np.unique(r[:, 0]):
            g = r[r[:, 0] == tag]
            spans.append((int(g[:, 4].min()), int(g[:, 6].max())))
            if kind == 1:  # the GEMM's shape rides in the kind word (gemm_ws.cu)
                w = int(g[0, 7])
                N, Kd, M, acc = ((w >> 8) & 0xFFFF) * 128, ((w >> 24) & 0xFFFF) * 64, (w >> 40) & 0xFFFF, (w >> 56) & 1
                stages = (w >> 57) & 7
                ctas, tiles = len(g), max(1, N // 128)
                per = -(-(Kd // 64) // max(1, ctas // tiles))
                pre = ctas * min(stages, per) * 128 * 64 * 2
                nbytes += Kd * N * 2 + M * Kd * 2 + M * N * 4 * (2 if acc else 1) - pre
            elif kind == 5:  # many-row tcgen05 GEMM: shape in the kind word (gemm_tc.cu)
                w = int(g[0, 7])
                N, Kd, M = ((w >> 8) & 0xFFFF) * 32, ((w >> 24) & 0xFFFF) * 64, (w >> 40) & 0xFFFF
                flops += 2 * M * N * Kd
                nbytes += Kd * N * 2 + M * Kd * 2 + M * N * 2
        spans.sort()
        busy, cur0, cur1 = 0, None, None
        for a, b in spans:
            if cur1 is None or a > cur1:
                if cur1 is not None:
                    busy += cur1 - cur0
                cur0, cur1 = a, b
            else:
                cur1 = max(cur1, b)
        busy += cur1 - cur0
        if kind == 2:
            nbytes = attn_step_bytes(be, m, prune_layer)
        elif kind == 1 and bonus_fused(be, m.batch):  # the bonus pass's attention runs in its QKV launches
            nbytes += bonus_attn_bytes(be, m)
        busy_ms = busy / 1e6
        gbs = nbytes / (busy_ms * 1e-3) / 1e9 if busy_ms > 0 else 0.0
        out[name] = {"launches": len(spans), "busy_ms": busy_ms, "bytes": nbytes, "achieved": gbs, "frac": gbs / hbm,
                     "share_of_step": busy_ms / out["step_ms"]}
        if kind == 5:  # tensor-bound at these row counts: TFLOP/s against the sustained bf16 peak
            tpk = tensor_peak()[0]
            tf = flops / (busy_ms * 1e-3) / 1e12 if busy_ms > 0 else 0.0
            out[name].update({"flops": flops, "tflops": tf, "tensor_frac": tf / tpk})
    return out


def prime_fn(be, eng, seqs, group, dev):
    def prime():
        # untimed: run until no new CUDA graph has been captured for 6
        # consecutive steps.  Under torchrun the decision is collective (every
        # rank runs the same number of steps: the steps contain a collective)
        stable, n = 0, 0
        while stable < 6 and n < 48:
            n_graphs = len(be._graphs)
            eng._step(seqs, 10 ** 9)
            n += 1
            changed = all_max(float(len(be._graphs) != n_graphs), group, dev)
            stable = stable + 1 if changed == 0.0 else 0
        return n
    return prime


def timed_steps(be, eng, seqs, K, group, dev):
    """K steps bracketed by a barrier + synchronize, CUDA events on the launch stream."""
    import torch

    torch.cuda.synchronize()
    if group is not None:
        torch.distributed.barrier(group)
    launches0, graphs0 = be.launches, len(be._graphs)
    stream = torch.cuda.current_stream(dev)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    metrics = []
    with ClockSampler(dev.index) as clk:
        t0.record(stream)
        for _ in range(K):
            metrics.append(eng._step(seqs, 10 ** 9))
        t1.record(stream)
        torch.cuda.synchronize()
        if group is not None:
            torch.distributed.barrier(group)
    return {"ms": all_max(t0.elapsed_time(t1), group, dev), "metrics": metrics, "clock": clk.summary(),
            "launches": be.launches - launches0, "captures": len(be._graphs) - graphs0}


class pinned_plan:
    """Within the block the engine keeps the tree plan `paths` (the plan of
    the timed steps: the dynamic plan may move afterwards, and the verify-ms,
    per-launch and traced-step measurements must see the same trees)."""

    def __init__(self, eng, paths):
        self.eng, self.paths = eng, paths

    def __enter__(self):
        if self.paths is not None:
            self.eng._plan = lambda batch, mean_seqlen: (self.paths, False)
        return self

    def __exit__(self, *exc):
        self.eng.__dict__.pop("_plan", None)
        return False


def verify_ms(be, eng, seqs, prime, K):
    """BASELINE's verify ms/step: two event nodes per step bracketing the tree
    pass (K1 -> layers -> K3 -> LM argmax -> K5) in otherwise unmodified graphs."""
    import torch

    be.attn_timer, be.mark_only = [], True
    try:
        prime()
        be.attn_timer = []
        for _ in range(K):
            eng._step(seqs, 10 ** 9)
        torch.cuda.synchronize()
        v = [r["ms"] for r in be.attn_timer if r.get("kind") == "verify"]
    finally:
        be.attn_timer, be.mark_only = None, False
    return sum(v) / max(1, len(v))


def run_b200(args, rank: int, world: int, group):
    import torch

    from paper_2402_13485_b200 import B200Backend, DecodeEngine
    from paper_2402_13485_b200.engine import _Seq

    dev = local_device(args)
    torch.cuda.set_device(dev)
    cfg = model_cfg(args)
    B = args.batch
    be = B200Backend(cfg, dtype="bf16", device=dev, random_device_init=True, max_slots=B + 1, max_tree=4 * args.topk,
                     kv_len=cfg.max_positions, attn_impl=args.attn_impl, use_graphs=not args.no_graphs)
    if args.planted:
        be.plant_draft_head(0)
    ecfg = engine_cfg(args)
    eng = DecodeEngine(be, ecfg, None, group=group)
    states = be.synthetic_states(B, args.kv, seed=1000 + rank)
    seqs = [_Seq(st, st.committed[:], rank * B + i) for i, st in enumerate(states)]
    if group is not None:  # the engine's multi-rank view of this synthetic batch
        from paper_2402_13485_b200.engine import _Global

        eng._glob = _Global([s.prompt for _ in range(world) for s in seqs], world)
    if args.sync_rows:
        be.device_rows = False
    prime = prime_fn(be, eng, seqs, group, dev)
    primed = prime()
    for _ in range(args.warmup):
        eng._step(seqs, 10 ** 9)
    be.attn_timer = None  # clean timed region: no per-launch event harvesting on the host
    main = timed_steps(be, eng, seqs, args.steps, group, dev)
    with pinned_plan(eng, eng._selection if ecfg.uses_dynamic else None):
        # second region of K steps: CUDA events around every K2 / GEMM launch
        # (event nodes inside separately captured graphs, each launch serialised)
        be.attn_timer = []
        prime()
        be.attn_timer = []
        for _ in range(args.steps):
            eng._step(seqs, 10 ** 9)
        torch.cuda.synchronize()
        events = be.attn_timer
        be.attn_timer = None
        vms = verify_ms(be, eng, seqs, prime, args.steps)
        prune_layer = ecfg.prune.layer if ecfg.uses_prune else None
        in_step = timeline_step(be, eng, seqs, prime, dev, prune_layer, modal_size(main["metrics"]))
    hbm, peak_kind = peaks()
    kernels = {}
    for kind in ("gemm", "attn", "gemm_tc"):
        rs = [r for r in events if r.get("kind", "attn") == kind]
        k_ms, k_bytes = sum(r["ms"] for r in rs), sum(r["bytes"] for r in rs)
        k_flops = sum(r.get("flops", 0) for r in rs)
        kernels[kind] = {"launches": len(rs), "ms_total": k_ms, "bytes": k_bytes, "flops": k_flops,
                         "achieved_gbs": k_bytes / (k_ms * 1e-3) / 1e9 if k_ms > 0 else 0.0,
                         "avg_launch_us": k_ms / max(1, len(rs)) * 1e3, "peak": hbm, "peak_kind": peak_kind}
    out = {"main": main, "kernels": kernels, "in_step": in_step, "verify_ms": vms, "priming_steps": primed,
           "streamed_bytes": be.w.streamed_bytes_per_step(prune=ecfg.uses_prune)}
    for st in states:  # free the synthetic sequences' cache slots for the e2e run
        be.release(st)
    eng._glob = None
    out["e2e"] = None if args.no_e2e else run_e2e(args, be, eng, rank, world, group)
    del be, eng, states, seqs
    torch.cuda.empty_cache()
    return out


def run_e2e(args, be, eng, rank, world, group):
    """End-to-end through the public API: DecodeEngine.run(prompts) from host
    token lists at the same KV length as `value` (H2D of the prompts, batched
    prefill, decode of 64 new tokens per sequence, per-step D2H of the step's
    results), wall clock, max over ranks."""
    import numpy as np
    import torch

    rng = np.random.default_rng(7)
    n_prompts = args.batch * world
    prompts = [rng.integers(0, be.V, size=args.kv).tolist() for _ in range(n_prompts)]
    max_tokens = 64
    eng.run([p[: args.kv] for p in prompts[:world]], 2, batch_size=world)  # warm path (prefill at this length)
    torch.cuda.synchronize()
    if group is not None:
        torch.distributed.barrier(group)
    graphs0 = len(be._graphs)
    t0 = time.perf_counter()
    res = eng.run(prompts, max_tokens, batch_size=n_prompts)
    torch.cuda.synchronize()
    dt = all_max(time.perf_counter() - t0, group, be.device)
    toks = sum(len(t) for t in res.transcripts)
    iters = max(1, res.summary.iterations)
    D, G = 4, 4 * args.topk
    hb = be._host.get((args.batch, D, G))
    d2h = sum(t.numel() * t.element_size() for t in hb.values()) if hb else 0
    return {"value": toks / dt, "unit": "tokens/s",
            "h2d_bytes_per_step": int(sum(len(p) for p in prompts) * 4 / iters),
            "d2h_bytes_per_step": int(d2h * world),
            "captures": len(be._graphs) - graphs0,
            "what": (f"DecodeEngine.run of {n_prompts} prompts x {args.kv} tokens (host lists), {max_tokens} new "
                     "tokens each, wall clock incl. H2D of the prompts, batched prefill, decode and the per-step D2H "
                     f"of each step's results ({iters} iterations)")}


def run_sweep(args, dev):
    """The north-star grid in this process (configs[2]; static tree vs ProPD at
    B=1, configs[1]): one backend sized for the largest point, a fresh synthetic
    batch per point; tok/s from a clean timed region, verify ms from the marker
    region, K2 / GEMM in-step roofline fractions from one traced step."""
    import torch

    from paper_2402_13485_b200 import B200Backend, DecodeEngine
    from paper_2402_13485_b200.engine import _Seq

    pts = []
    for spec in args.sweep_points.split(","):
        f = spec.split(":")
        pts.append((int(f[0]), int(f[1]), f[2] if len(f) > 2 else "propd_full"))
    K = 5
    kv_max, b_max = max(p[1] for p in pts), max(p[0] for p in pts)
    # per point: <= 3 priming phases of <= 48 steps + K + 3 + 1 steps of ~1 token (random init)
    margin = 2 * (3 * 48 + K + 4) + 16
    cfg = model_cfg(args, kv_cap=kv_max)
    cfg = type(cfg)(**{**cfg.__dict__, "max_positions": kv_max + margin})
    be = B200Backend(cfg, dtype="bf16", device=dev, random_device_init=True, max_slots=b_max,
                     max_tree=4 * args.topk, kv_len=cfg.max_positions, use_graphs=True)
    rows = []
    for B, kv, mode in pts:
        t_start = time.perf_counter()
        row = {"batch": B, "kv": kv, "mode": mode}
        try:
            ecfg = engine_cfg(args, mode)
            eng = DecodeEngine(be, ecfg, None)
            states = be.synthetic_states(B, kv, seed=B * 7919 + kv)
            seqs = [_Seq(st, st.committed[:], i) for i, st in enumerate(states)]
            prime = prime_fn(be, eng, seqs, None, dev)
            prime()
            r = timed_steps(be, eng, seqs, K, None, dev)
            m = r["metrics"]
            with pinned_plan(eng, eng._selection if ecfg.uses_dynamic else None):
                vms = verify_ms(be, eng, seqs, prime, 3)
                ins = timeline_step(be, eng, seqs, prime, dev, ecfg.prune.layer if ecfg.uses_prune else None,
                                    modal_size(m))
            row.update({"tok_s": sum(x.tokens_committed for x in m) / (r["ms"] * 1e-3), "ms_per_step": r["ms"] / K,
                        "verify_ms_per_step": vms, "accepted_len_per_step": sum(x.mean_accepted for x in m) / K,
                        "tree_size_mean": sum(x.tree_size for x in m) / K,
                        "traced_tree_size": ins.get("traced_tree_size"),
                        "k2_frac_in_step": ins.get("attn", {}).get("frac"),
                        "gemm_frac_in_step": ins.get("gemm", {}).get("frac"),
                        "gemm_tc_tensor_frac_in_step": ins.get("gemm_tc", {}).get("tensor_frac"),
                        "k2_share_of_step": ins.get("attn", {}).get("share_of_step"),
                        "clocks": r["clock"], "captures_in_timed_region": r["captures"]})
            for st in states:
                be.release(st)
        except Exception as exc:  # a point that does not fit is reported, not fatal
            row["error"] = f"{type(exc).__name__}: {exc}"[:200]
            torch.cuda.synchronize()
        row["wall_s"] = round(time.perf_counter() - t_start, 1)
        rows.append(row)
    del be
    torch.cuda.empty_cache()
    return {"points": rows, "steps_per_point": K,
            "note": ("B200 arm, same process and kernels as `value`: 7B shape, random init, tok/s = committed tokens / "
                     "device time of 5 steps after graph priming; K2 / GEMM fractions of the measured copy peak inside "
                     "one traced step (union of [dependency release, last CTA exit] per launch); static_tree = the "
                     "full 64-node Medusa grid without pruning")}


def roofline(res, args) -> dict:
    """Roofline of the kernel family with the largest busy share of the traced step."""
    ins = res["in_step"]
    fam = {k: v for k, v in ins.items() if isinstance(v, dict)}
    dom = max(fam, key=lambda k: fam[k]["busy_ms"])
    d = fam[dom]
    hbm, peak_kind = peaks()
    ev = res["kernels"].get(dom, {})
    names = {"gemm": "weight-streaming tcgen05 projections (propd_gemm_ws, <= 128 rows)",
             "attn": "K2 tree-masked verification attention (tcgen05 tcT / tc2 kernels + streaming decode kernel)",
             "gemm_tc": "many-row tcgen05 projections (propd_gemm, > 128 rows)"}
    if dom == "gemm_tc":
        tpk, tburst, tkind = tensor_peak()
        return {"kernel": names[dom], "bound": "tensor", "achieved": d["tflops"], "peak": tpk, "unit": "TFLOP/s",
                "frac": d["tflops"] / tpk, "burst_peak": tburst, "traffic": ncu_traffic(dom, args).get("bytes_per_launch"),
                "peak_kind": tkind, "launches_per_step": d["launches"], "share_of_step": d["share_of_step"],
                "algorithmic_flops_per_step": d["flops"],
                "timer": "device globaltimer per CTA: union of [dependency release, last CTA exit] per launch, one step"}
    out = {"kernel": names[dom], "bound": "hbm", "achieved": d["achieved"], "peak": hbm, "unit": "GB/s",
           "frac": d["achieved"] / hbm, "traffic": ncu_traffic(dom, args).get("bytes_per_launch"),
           "traffic_note": ncu_traffic(dom, args).get("note"), "peak_kind": peak_kind,
           "launches_per_step": d["launches"], "avg_launch_us": d["busy_ms"] * 1e3 / max(1, d["launches"]),
           "share_of_step": d["share_of_step"],
           "algorithmic_bytes_per_step": d["bytes"],
           "timer": "device globaltimer per CTA: union of [dependency release, last CTA exit] per launch, one step"}
    if ev.get("launches"):
        out["events_achieved"] = ev["achieved_gbs"]
        out["events_frac"] = ev["achieved_gbs"] / hbm
        out["events_avg_launch_us"] = ev["avg_launch_us"]
        out["events_note"] = "CUDA events around each launch (serialises the PDL chain; ramp included)"
    return out


def reference_line(args):
    ref = cpu_reference(args, args.steps, args.warmup, [int(x) for x in args.ref_tree_sizes.split(",")])
    return {"metric": METRIC, "value": ref["value"], "unit": "tokens/s", "n_gpus": args.gpus, "steps": ref["steps"],
            "warmup": args.warmup, "ms_per_step": ref["ms_per_step"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (random-init weights and prompts)",
            "impl": "reference",
            "config": config_block(args, 1),
            "accepted_len_per_step": ref["accepted_len_per_step"], "tree_size_mean": ref["tree_size_mean"],
            "cpu_baseline": {k: ref[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": ref["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def config_block(args, world):
    shape7 = args.shape == "7b"
    return {"workload": ("configs[1]: Vicuna-7B-shape" if shape7 else "configs[3]: Vicuna-33B-shape")
                        + f" random-init bf16, batch {args.batch}/GPU, KV {args.kv}, {args.mode}"
                        + (", planted draft head 0 (accepts depth-1 nodes)" if args.planted else ""),
            "model": ("vicuna-7b-shape (32L, 4096, 32x128, V32000, 4 draft heads)" if shape7
                      else "vicuna-33b-shape (60L, 6656, 52x128, V32000, 4 draft heads)"),
            "batch_per_gpu": args.batch, "global_batch": args.batch * world, "kv": args.kv, "mode": args.mode,
            "draft_topk": args.topk,
            "prune": ("layer 4, top-K 50" if args.prune_threshold is None
                      else f"layer 4, path probability >= {args.prune_threshold}"),
            "acceptance": args.acceptance, "parallelism": f"dp{world} (sequence-sharded replicas)",
            "l2": "inputs larger than L2 (14.8 GB of weights stream twice per step)"}


def relaunch(args) -> int:
    """--gpus N > 1 outside torchrun: run this script under torchrun, one rank per GPU."""
    import random

    port = str(29600 + random.randint(0, 3000))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        if rank == 0:  # the CPU path: rank 0 alone, every host thread
            print(json.dumps(reference_line(args)))
        return
    group = None
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_device(args))
        dist.init_process_group(args.dist_backend)
        group = dist.group.WORLD
    res = run_b200(args, rank, world, group)
    sweep = None
    if world == 1 and not args.no_sweep:
        sweep = run_sweep(args, local_device(args))
    if rank != 0:
        if group is not None:
            import torch.distributed as dist

            dist.destroy_process_group()
        return
    main_r = res["main"]
    m, ms, K = main_r["metrics"], main_r["ms"], args.steps
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        try:  # the reference arm's measurement on this arm's own tree-size schedule
            steps = min(K, 4)
            c = cpu_reference(args, steps, 1, [x.tree_size for x in m[:steps]])
            cpu = {k: c[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as exc:  # pragma: no cover
            cpu = {"value": None, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"failed: {exc}"}
    kern = res["kernels"]
    line = {
        "metric": METRIC,
        "value": main_r["metrics"] and sum(x.tokens_committed for x in m) / (ms * 1e-3),
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": K,
        "warmup": args.warmup,
        "ms_per_step": ms / K,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (random-init weights, random KV/prompt state)",
        "config": config_block(args, world),
        "accepted_len_per_step": sum(x.mean_accepted for x in m) / K,
        "tree_size_mean": sum(x.tree_size for x in m) / K,
        "tree_sizes": [x.tree_size for x in m],
        "prune_rate_mean": sum(x.prune_rate for x in m) / K,
        "verify_ms_per_step": res["verify_ms"],
        "verify_ms_note": ("tree pass K1 -> layers -> K3 -> LM argmax -> K5 (excludes draft heads and the bonus pass): "
                           "two CUDA event nodes per step in otherwise unmodified graphs, mean over K steps"),
        "roofline": roofline(res, args),
        "roofline_by_kernel": {k: {"achieved": v["achieved_gbs"], "frac": v["achieved_gbs"] / v["peak"],
                                   "tflops": (v["flops"] / (v["ms_total"] * 1e-3) / 1e12) if v["ms_total"] > 0 else 0.0,
                                   "ms_per_step": v["ms_total"] / K, "launches_per_step": v["launches"] / K,
                                   "avg_launch_us": v["avg_launch_us"]} for k, v in kern.items()},
        "in_step": res["in_step"],
        "step_weight_gbs": res["streamed_bytes"] / (ms / K * 1e-3) / 1e9,
        "step_weight_note": ("weight bytes streamed per step (layers + LM head twice, early head, draft heads; the "
                             "embedding / position tables are gathered) / ms_per_step"),
        "gpu_launches": main_r["launches"],
        "cuda_graphs": {"priming_steps": res["priming_steps"], "captures_in_timed_region": main_r["captures"]},
        "clocks": main_r["clock"],
        "cpu_baseline": cpu,
        "e2e": res["e2e"],
        "sweep": sweep,
    }
    print(json.dumps(line))
    if group is not None:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
