"""Per-launch view of one traced bench step (development aid): reads the raw
per-CTA records bench.py saves with PROPD_BENCH_DUMP=path.npy and prints, per
kernel family and shape, launches, mean window (dependency release -> last
CTA exit), mean gap to the previous launch's exit, and the sum of windows.

  PROPD_BENCH_DUMP=gpurun_out/rec.npy python bench.py --no-sweep ...
  python scripts/step_records.py gpurun_out/rec.npy
"""
import sys
from collections import defaultdict

import numpy as np

rec = np.load(sys.argv[1])
tags = np.unique(rec[:, 0])
rows = []
for tg in tags:
    g = rec[rec[:, 0] == tg]
    kind = int(g[0, 7]) & 0xFF
    w = int(g[0, 7])
    if kind == 1:
        N, K, M = ((w >> 8) & 0xFFFF) * 128, ((w >> 24) & 0xFFFF) * 64, (w >> 40) & 0xFFFF
        name = f"gws N={N} K={K} M={M}"
    elif kind == 5:
        N, K, M = ((w >> 8) & 0xFFFF) * 32, ((w >> 24) & 0xFFFF) * 64, (w >> 40) & 0xFFFF
        name = f"gtc N={N} K={K} M={M}"
    else:
        name = {2: "attn", 4: "attn_tct"}.get(kind, f"kind{kind}") + f" ctas={len(g)}"
    rows.append((int(g[:, 4].min()), int(g[:, 4].max()), int(g[:, 6].max()), name))
rows.sort()
agg = defaultdict(lambda: [0, 0.0, 0.0])
prev_exit = None
for rel0, rel1, ex, name in rows:
    a = agg[name]
    a[0] += 1
    a[1] += (ex - rel1) / 1e3
    a[2] += ((rel1 - prev_exit) / 1e3) if prev_exit is not None else 0.0
    prev_exit = ex
total = (rows[-1][2] - rows[0][0]) / 1e3
win_all = sum(a[1] for a in agg.values())
gap_all = sum(a[2] for a in agg.values())
print(f"{len(rows)} traced launches, span {total:.1f} us: windows {win_all:.1f} us, gaps before releases {gap_all:.1f} us")
for name, (n, win, gap) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{name:34s} x{n:4d}  window {win / n:7.2f} us  gap {gap / n:6.2f} us  sum {win:8.1f} us")
