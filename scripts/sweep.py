"""Batch x KV sweep (BASELINE configs[2] / [3]): one bench.py run per point,
a markdown table of tok/s, ms/step, verify ms/step and the in-step roofline
fractions of the two kernel families.

  python scripts/sweep.py --shape 7b --batches 1,8,16,32,64 --kvs 512,1024,2048,4096 --out gpurun_out/sweep.md
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="7b")
ap.add_argument("--batches", default="1,8,16,32,64")
ap.add_argument("--kvs", default="512,1024,2048,4096")
ap.add_argument("--points", default="", help="explicit B:KV list (overrides --batches/--kvs)")
ap.add_argument("--out", default="gpurun_out/sweep.md")
args = ap.parse_args()
if args.points:
    points = [tuple(map(int, p.split(":"))) for p in args.points.split(",")]
else:
    points = [(b, kv) for b in map(int, args.batches.split(",")) for kv in map(int, args.kvs.split(","))]
rows = []
for B, kv in points:
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--shape", args.shape, "--batch", str(B), "--kv", str(kv),
           "--steps", "10", "--no-e2e", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=ROOT)
    try:
        d = json.loads(r.stdout.strip().splitlines()[-1])
    except Exception:
        rows.append(f"| {B} | {kv} | failed: {(r.stderr or r.stdout)[-160:]!r} |")
        print(rows[-1], flush=True)
        continue
    ins = d.get("in_step", {})
    frac = lambda k: f"{ins[k]['frac']:.2f}" if isinstance(ins.get(k), dict) else "-"
    cap = d.get("cuda_graphs", {}).get("captures_in_timed_region", 0)
    rows.append(f"| {B} | {kv} | {d['value']:.1f} | {d['ms_per_step']:.2f} | {d.get('verify_ms_per_step', 0):.2f} | "
                f"{d.get('tree_size_mean', 0):.1f} | {frac('gemm')} | {frac('attn')} | "
                f"{d['clocks']['sm_mhz']:.0f} {','.join(d['clocks']['reasons'])} | {cap} |")
    print(rows[-1], flush=True)
hdr = ("| batch | KV | tok/s | ms/step | verify ms/step | mean tree size | GEMM frac (in-step) | K2 frac (in-step) | "
       "SM MHz, throttle | graph captures in timed steps |\n|---|---|---|---|---|---|---|---|---|---|\n")
with open(os.path.join(ROOT, args.out), "w") as fh:
    fh.write(hdr + "\n".join(rows) + "\n")
