"""Per-step GPU vs host timeline of the bench workload (development aid):
CUDA events around every graph replay + host perf counters, no profiler."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2402_13485_b200 import B200Backend, DecodeEngine  # noqa: E402
from paper_2402_13485_b200.engine import _Seq  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--kv", type=int, default=1024)
ap.add_argument("--layers", type=int, default=32)
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--mode", default="propd_full")
ap.add_argument("--topk", type=int, default=16)
args = ap.parse_args()

cfg = bench.model_cfg(args)
be = B200Backend(cfg, dtype="bf16", random_device_init=True, max_slots=args.batch + 1, kv_len=cfg.max_positions,
                 use_graphs=True)
eng = DecodeEngine(be, bench.engine_cfg(args), None)
states = be.synthetic_states(args.batch, args.kv)
seqs = [_Seq(st, st.committed[:], i) for i, st in enumerate(states)]
for _ in range(40):
    eng._step(seqs, 10 ** 9)
torch.cuda.synchronize()

log = []
orig = be._run


def run(key, fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    out = orig(key, fn)
    e1.record()
    t1 = time.perf_counter()
    log.append((key[0], e0, e1, t0, t1))
    return out


be._run = run
s0 = torch.cuda.Event(enable_timing=True)
s0.record()
t_start = time.perf_counter()
for _ in range(args.steps):
    eng._step(seqs, 10 ** 9)
torch.cuda.synchronize()
wall = (time.perf_counter() - t_start) * 1e3 / args.steps
gpu = {}
launch = {}
for name, e0, e1, t0, t1 in log:
    gpu[name] = gpu.get(name, 0.0) + e0.elapsed_time(e1)
    launch[name] = launch.get(name, 0.0) + (t1 - t0) * 1e3
first = log[0][1]
span = first.elapsed_time(log[-1][2]) / args.steps
print(f"wall {wall:.3f} ms/step; device span {span:.3f} ms/step")
for k in gpu:
    print(f"  graph {k}: gpu {gpu[k] / args.steps:.3f} ms/step, host replay call {launch[k] / args.steps * 1e3:.1f} us/step")
# gaps between consecutive graphs
gaps = [log[i][1].elapsed_time(log[i + 1][1]) - log[i][1].elapsed_time(log[i][2]) for i in range(len(log) - 1)]
print(f"  sum of inter-graph gaps {sum(gaps) / args.steps * 1e3:.1f} us/step")
