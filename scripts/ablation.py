"""Ablation sweep (BASELINE configs[4]): engine mode x batch x draft top-k at
the 7B shape, one bench.py run each; writes a markdown table.

  python scripts/ablation.py --out gpurun_out/ablation.md
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ap = argparse.ArgumentParser()
ap.add_argument("--out", default="gpurun_out/ablation.md")
ap.add_argument("--batches", default="1,16")
ap.add_argument("--topks", default="4,16,64")
ap.add_argument("--modes", default="static_tree,prune_only,dynamic_only,propd_full,autoregressive")
ap.add_argument("--kv", type=int, default=1024)
args = ap.parse_args()
rows = []
for B in map(int, args.batches.split(",")):
    for k in map(int, args.topks.split(",")):
        for mode in args.modes.split(","):
            if mode == "autoregressive" and k != int(args.topks.split(",")[0]):
                continue
            cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--batch", str(B), "--kv", str(args.kv), "--topk",
                   str(k), "--mode", mode, "--steps", "5", "--no-e2e", "--no-cpu-baseline"]
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
            try:
                d = json.loads(r.stdout.strip().splitlines()[-1])
            except Exception:
                rows.append(f"| {mode} | {B} | {k} | failed: {(r.stderr or r.stdout)[-200:]!r} |")
                continue
            rows.append(f"| {mode} | {B} | {4 * k} | {d['value']:.1f} | {d['ms_per_step']:.2f} | "
                        f"{d.get('verify_ms_per_step', 0):.2f} | {d['tree_size_mean']:.1f} | {d['prune_rate_mean']:.2f} | "
                        f"{d['roofline']['frac']:.2f} |")
            print(rows[-1], flush=True)
hdr = ("| mode | batch | grid nodes (4 x top-k) | tok/s | ms/step | verify ms/step | mean tree size | prune rate | "
       "dominant-kernel roofline frac |\n|---|---|---|---|---|---|---|---|---|\n")
with open(os.path.join(ROOT, args.out), "w") as fh:
    fh.write(hdr + "\n".join(rows) + "\n")
