"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv
--log-file X.csv python bench.py ...`) per engine step: the list is cut into
steps at every `stats_replay_select_kernel` launch (one per step, the last
kernel of the step) and the last --steps steps are averaged per kernel name.

  python scripts/ncu_launch_summary.py gpurun_out/launches.csv --steps 4 [--out profiles/x.csv]
"""
import argparse
import csv
import io
import sys

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--out")
ap.add_argument("--title", default="")
args = ap.parse_args()

text = open(args.csv).read()
start = text.find('"ID"')
rows = list(csv.DictReader(io.StringIO(text[start:])))
launches = []
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    unit = r.get("Metric Unit", "ns")
    v = float(r["Metric Value"].replace(",", ""))
    v *= {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
    launches.append((r["Kernel Name"], v))
cuts = [i for i, (k, _) in enumerate(launches) if "stats_replay_select" in k]
if len(cuts) < args.steps + 1:
    sys.exit(f"only {len(cuts)} step boundaries in {len(launches)} launches")
sel = launches[cuts[-args.steps - 1] + 1: cuts[-1] + 1]
agg: dict = {}
for k, v in sel:
    t, c = agg.get(k, (0.0, 0))
    agg[k] = (t + v, c + 1)
total = sum(t for t, _ in agg.values())
out = io.StringIO()
if args.title:
    out.write(f"# {args.title}\n")
out.write(f"# ncu launch list, last {args.steps} steps; serialised, cold-cache per launch\n")
out.write(f"# GPU kernel time per step: {total / args.steps:.3f} ms over {len(sel) / args.steps:.0f} launches\n")
out.write("ms_per_step,launches_per_step,share,avg_us,kernel\n")
for k, (t, c) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    out.write(f"{t / args.steps:.4f},{c / args.steps:.1f},{t / total:.3f},{t / c * 1e3:.2f},{k[:70]}\n")
print(out.getvalue())
if args.out:
    open(args.out, "w").write(out.getvalue())
