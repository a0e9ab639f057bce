"""Break one bench step into host phases (development aid)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import argparse  # noqa: E402

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2402_13485_b200 import B200Backend, DecodeEngine  # noqa: E402
from paper_2402_13485_b200 import backend as bk  # noqa: E402
from paper_2402_13485_b200.engine import _Seq  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--kv", type=int, default=1024)
ap.add_argument("--layers", type=int, default=32)
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--mode", default="propd_full")
ap.add_argument("--topk", type=int, default=16)
ap.add_argument("--attn-impl", type=int, default=0)
args = ap.parse_args()
cfg = bench.model_cfg(args)
be = B200Backend(cfg, dtype="bf16", random_device_init=True, max_slots=args.batch + 1, kv_len=cfg.max_positions,
                 max_tree=4 * args.topk, use_graphs=True)
eng = DecodeEngine(be, bench.engine_cfg(args), None)
seqs = [_Seq(st, st.committed[:], i) for i, st in enumerate(be.synthetic_states(args.batch, args.kv))]
for _ in range(20):
    eng._step(seqs, 10 ** 9)
if os.environ.get("GC_FREEZE") == "1":
    import gc
    gc.collect()
    gc.freeze()
T = {}
orig_run, orig_item = be._run, torch.Tensor.item


def timed(name, fn):
    def w(*a, **k):
        t0 = time.perf_counter()
        r = fn(*a, **k)
        T[name] = T.get(name, 0.0) + time.perf_counter() - t0
        return r
    return w


be._run = timed("graph_replay_calls", be._run)
be._slot_buf = timed("slot_buf", be._slot_buf)
be._harvest = timed("harvest", be._harvest)
be._host_bufs = timed("host_bufs", be._host_bufs)
torch.Tensor.item = timed("item_sync", orig_item)
be.step_tree = timed("step_tree_total", be.step_tree)
eng._plan = timed("plan", eng._plan)
torch.cuda.synchronize()
t0 = time.perf_counter()
per = []
for _ in range(args.steps):
    ts = time.perf_counter()
    ng = len(be._graphs)
    m = eng._step(seqs, 10 ** 9)
    per.append((time.perf_counter() - ts, m.replanned, m.tree_size, len(be._graphs) - ng, m.mean_survivors))
torch.cuda.synchronize()
wall = time.perf_counter() - t0
for i, (dt, rp, ts_, ng, sv) in enumerate(per):
    print(f"step {i}: {dt * 1e3:6.2f} ms replanned={rp} tree={ts_} new_graphs={ng} surv={sv}")
torch.Tensor.item = orig_item
print(f"wall {wall / args.steps * 1e3:.2f} ms/step")
if os.environ.get("PROFILE_PLAN") == "1":
    import cProfile
    import pstats
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(args.steps):
        eng._step(seqs, 10 ** 9)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
for k, v in sorted(T.items(), key=lambda kv: -kv[1]):
    print(f"  {k:22s} {v / args.steps * 1e3:7.3f} ms/step")
