"""Profile a few bench steps with torch.profiler (CPU + CUDA) — development aid.

  python scripts/profile_step.py --batch 1 --kv 1024 --layers 32 [--attn-impl 0]
"""
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
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--mode", default="propd_full")
ap.add_argument("--topk", type=int, default=16)
ap.add_argument("--attn-impl", type=int, default=0)
ap.add_argument("--out", default="gpurun_out/profile")
ap.add_argument("--graphs", action="store_true")
ap.add_argument("--no-cpu-baseline", action="store_true")
args = ap.parse_args()

cfg = bench.model_cfg(args)
be = B200Backend(cfg, dtype="bf16", random_device_init=True, max_slots=args.batch + 1, kv_len=cfg.max_positions,
                 attn_impl=args.attn_impl, use_graphs=args.graphs)
eng = DecodeEngine(be, bench.engine_cfg(args), None)
states = be.synthetic_states(args.batch, args.kv)
seqs = [_Seq(st, st.committed[:], i) for i, st in enumerate(states)]
for _ in range(len(eng._probe_queue) + 1 + args.warmup):
    eng._step(seqs, 10 ** 9)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(args.steps):
    eng._step(seqs, 10 ** 9)
torch.cuda.synchronize()
print(f"plain: {(time.perf_counter() - t0) / args.steps * 1e3:.2f} ms/step")
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(args.steps):
        eng._step(seqs, 10 ** 9)
    torch.cuda.synchronize()
os.makedirs(os.path.dirname(args.out), exist_ok=True)
ka = prof.key_averages()
with open(args.out + "_cuda.txt", "w") as fh:
    fh.write(ka.table(sort_by="cuda_time_total", row_limit=40))
with open(args.out + "_cpu.txt", "w") as fh:
    fh.write(ka.table(sort_by="self_cpu_time_total", row_limit=40))
print(ka.table(sort_by="cuda_time_total", row_limit=25))
print(ka.table(sort_by="self_cpu_time_total", row_limit=25))
