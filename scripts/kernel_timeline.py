"""Per-CTA globaltimer timeline of the per-layer kernels (development aid).

Runs --layers blocks over --rows tree rows at KV --kv eagerly (PDL chain as in
the product path, no graph), with the libpropd trace buffer installed
(propd_debug_timeline; instrumented kernels: weight-streaming GEMM, tc2 and
decode attention).  Prints, per traced launch, relative to the first entry:
first CTA entry, last pdl-wait release, last main-loop end, last exit.

  python scripts/kernel_timeline.py --rows 16 --kv 1024 --layers 4 [--unfused]
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2402_13485_b200 import B200Backend, TinyTransformerConfig, _lib  # noqa: E402
from paper_2402_13485_b200.backend import Rows  # noqa: E402
from paper_2402_13485_b200.tree import TreeTemplate  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=16)
ap.add_argument("--kv", type=int, default=1024)
ap.add_argument("--layers", type=int, default=4)
ap.add_argument("--show", type=int, default=2, help="layers to print")
ap.add_argument("--unfused", action="store_true")
ap.add_argument("--per-cta", action="store_true", help="attention: per-CTA phase percentiles")
ap.add_argument("--dump", default=None, help="save the raw CTA records (.npy)")
args = ap.parse_args()

cfg = TinyTransformerConfig(layers=args.layers, hidden=4096, heads=32, vocab=32000, draft_heads=4,
                            max_positions=args.kv + 256, seed=0)
be = B200Backend(cfg, dtype="bf16", random_device_init=True, max_slots=2, max_tree=64, kv_len=cfg.max_positions)
be.ws_phases = not args.unfused
states = be.synthetic_states(1, args.kv)
dev = be.device
paths = sorted({(1,) * d for d in range(1, 5)} | {(r,) for r in range(1, 17)} | {(1, r) for r in range(1, 17)})
tmpl = TreeTemplate.from_paths(paths[:args.rows] if len(paths) >= args.rows else paths)
n = len(tmpl)
td = tmpl.device(dev)
i32 = lambda a: torch.tensor(a, device=dev, dtype=torch.int32)
rt = Rows(n, 1, i32([states[0].slot]), i32([0] * n), i32(list(range(n))), i32([0, n]), max_keys=args.kv + n + 8,
          max_rows=n)
x = torch.randn(n, 4096, device=dev)
lib = _lib.load()
for _ in range(3):
    be._run_layers(x.clone(), rt, 0, args.layers, td["mask"], n, tmpl.words)
torch.cuda.synchronize()
buf = torch.zeros(8 + 8 * 200000, device=dev, dtype=torch.int64)
buf[1] = 200000
lib.propd_debug_timeline(ctypes.c_void_p(buf.data_ptr()))
be._run_layers(x.clone(), rt, 0, args.layers, td["mask"], n, tmpl.words)
torch.cuda.synchronize()
lib.propd_debug_timeline(ctypes.c_void_p(0))
cnt = int(buf[0].item())
rec = buf[8: 8 + 8 * cnt].view(cnt, 8).cpu().numpy().astype(np.int64)
t_ref = rec[:, 3].min()
if args.dump:
    np.save(args.dump, rec)
print(f"rows {n}, kv {args.kv}, {'unfused' if args.unfused else 'fused'}: {cnt} CTA records")
print(f"{'tag':>4} {'ctas':>5} {'entry0':>8} {'entry1':>8} {'wait_max':>8} {'main_max':>8} {'exit_min':>8} "
      f"{'exit_max':>8} {'gap':>6}  (us)")
prev_exit = None
per_layer = None
tags = sorted(set(rec[:, 0].tolist()))
for tg in tags:
    r = rec[rec[:, 0] == tg]
    us = lambda v: (v - t_ref) / 1e3
    gap = us(r[:, 4].max()) - prev_exit if prev_exit is not None else 0.0
    print(f"{tg:4d} {len(r):5d} {us(r[:, 3].min()):8.1f} {us(r[:, 3].max()):8.1f} {us(r[:, 4].max()):8.1f} "
          f"{us(r[:, 5].max()):8.1f} {us(r[:, 6].min()):8.1f} {us(r[:, 6].max()):8.1f} {gap:6.1f}")
    prev_exit = us(r[:, 6].max())
    if args.per_cta and r[0, 7] == 4:  # tcT: records (first S, wait, loop end, exit)
        q = lambda v: " ".join(f"{x:5.2f}" for x in np.percentile(v / 1e3, [0, 50, 90, 100]))
        print(f"      tcT per-CTA [p0 p50 p90 max] wait->S0 {q(r[:, 3] - r[:, 4])}  S0->loop end {q(r[:, 5] - r[:, 3])}"
              f"  ->exit {q(r[:, 6] - r[:, 5])}")
    if args.per_cta and r[0, 7] == 2:  # attention: per-CTA wait -> loop end -> exit
        q = lambda v: " ".join(f"{x:5.2f}" for x in np.percentile(v / 1e3, [0, 50, 90, 100]))
        print(f"      per-CTA wait->main [p0 p50 p90 max] {q(r[:, 5] - r[:, 4])}   main->exit {q(r[:, 6] - r[:, 5])}")
span = (rec[:, 6].max() - t_ref) / 1e3
print(f"span {span:.1f} us for {args.layers} layers = {span / args.layers:.1f} us/layer")
