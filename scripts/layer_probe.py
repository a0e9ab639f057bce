"""Time the weight-streaming layer stack at 7B width for a few rows, with
parts of each layer switched off (development aid): where does a layer's
time go beyond its 403 MB weight stream?

  python scripts/layer_probe.py --rows 16 --kv 1024 --layers 8
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2402_13485_b200 import B200Backend, TinyTransformerConfig  # noqa: E402
from paper_2402_13485_b200.backend import Rows  # noqa: E402
from paper_2402_13485_b200.tree import TreeTemplate  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=16)
ap.add_argument("--kv", type=int, default=1024)
ap.add_argument("--layers", type=int, default=8)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--unfused", action="store_true")
args = ap.parse_args()

cfg = TinyTransformerConfig(layers=args.layers, hidden=4096, heads=32, vocab=32000, draft_heads=4,
                            max_positions=args.kv + 256, seed=0)
be = B200Backend(cfg, dtype="bf16", random_device_init=True, max_slots=2, max_tree=64, kv_len=cfg.max_positions,
                 use_graphs=True)
states = be.synthetic_states(1, args.kv)
dev = be.device
n = args.rows
paths = sorted({(1,) * d for d in range(1, 5)} | {(r,) for r in range(1, 17)} | {(1, r) for r in range(1, 17)})
tmpl = TreeTemplate.from_paths(paths[:n] if len(paths) >= n else paths)
n = len(tmpl)
td = tmpl.device(dev)
i32 = lambda a: torch.tensor(a, device=dev, dtype=torch.int32)
rt = Rows(n, 1, i32([states[0].slot]), i32([0] * n), i32(list(range(n))), i32([0, n]), max_keys=args.kv + n + 8,
          max_rows=n)
x = torch.randn(n, 4096, device=dev)
orig_call = be._call


def run(skip):
    def call(name, *a):
        if name in skip:
            return
        return orig_call(name, *a)

    be._call = call
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        be._run_layers(x, rt, 0, args.layers, td["mask"], n, tmpl.words)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        be._run_layers(x, rt, 0, args.layers, td["mask"], n, tmpl.words)
    be._call = orig_call
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / args.reps / args.layers


floor = 402653184 / 6543.1e9 * 1e6
print(f"rows {n}, kv {args.kv}: weight floor {floor:.1f} us/layer")
if "--unfused" in sys.argv:
    be.ws_phases = False
for label, skip in [("full layer", set()), ("no attention", {"propd_tree_attention"}),
                    ("no add_ln", {"propd_add_ln"}), ("no finish", {"propd_qkv_finish", "propd_gelu_finish"}),
                    ("GEMMs only", {"propd_tree_attention", "propd_add_ln", "propd_qkv_finish", "propd_gelu_finish"})]:
    print(f"  {label:14s} {run(skip):7.1f} us/layer")
