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
ap.add_argument("--sync-rows", action="store_true", help="size the post-prune pass on the host (mid-step sync)")
args = ap.parse_args()

cfg = bench.model_cfg(args)
be = B200Backend(cfg, dtype="bf16", random_device_init=True, max_slots=args.batch + 1, kv_len=cfg.max_positions,
                 attn_impl=args.attn_impl, use_graphs=args.graphs)
be.device_rows = not args.sync_rows
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

# GPU idle gaps between consecutive device activities (kernels + memcpys)
import json  # noqa: E402

prof.export_chrome_trace(args.out + "_trace.json")
ev = [e for e in json.load(open(args.out + "_trace.json"))["traceEvents"]
      if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
gaps = []
for a_, b_ in zip(ev, ev[1:]):
    g = b_["ts"] - (a_["ts"] + a_["dur"])
    gaps.append((g, a_["name"][:50], b_["name"][:50]))
span = ev[-1]["ts"] + ev[-1]["dur"] - ev[0]["ts"]
busy = sum(e["dur"] for e in ev)
print(f"device span {span / args.steps:.1f} us/step, busy {busy / args.steps:.1f} us/step, "
      f"{len(ev) / args.steps:.0f} activities/step, gaps<=3us sum {sum(g for g, _, _ in gaps if g <= 3) / args.steps:.1f}"
      f" us/step, gaps>3us sum {sum(g for g, _, _ in gaps if g > 3) / args.steps:.1f} us/step")
for g, a_, b_ in sorted(gaps, reverse=True)[:12]:
    print(f"  gap {g:8.1f} us  after {a_}  before {b_}")
