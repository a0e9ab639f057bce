"""Throughput of K2 alone (development aid): 20 back-to-back launches of the
tree-pass kernel (rows per sequence = --rows, tc2 / auto) and of the decode
kernel (1 row) in a CUDA graph, at 7B head geometry (32 x 128), over
--batch sequences of KV length --kv.  Prints achieved GB/s of algorithmic
bytes (K/V rows + Q + O) against the measured copy bandwidth.

  python scripts/attn_probe.py --batch 64 --kv 4096 --rows 20
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2402_13485_b200 import _lib  # noqa: E402
from paper_2402_13485_b200._lib import call, ptr  # noqa: E402
from paper_2402_13485_b200.tree import TreeTemplate  # noqa: E402
from oracle import treedecode_port as op  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--kv", type=int, default=4096)
ap.add_argument("--rows", type=int, default=20)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--impl", type=int, default=0)
ap.add_argument("--cap", type=int, default=0, help="row capacity passed as max_rows_per_seq (default: --rows)")
args = ap.parse_args()

dev = torch.device("cuda:0")
A, dh = 32, 128
H = A * dh
B, L = args.batch, args.kv
tmpl = TreeTemplate.from_paths(op.grid_candidates(4, 16))  # 64-node template; rows = first args.rows nodes
n = len(tmpl)
Lmax = L + n + 8
kc = torch.randn(B, A, Lmax, dh, device=dev).bfloat16()
vc = torch.randn(B, A, Lmax, dh, device=dev).bfloat16()
lens = torch.full((B,), L, dtype=torch.int32, device=dev)
slots = torch.arange(B, dtype=torch.int32, device=dev)
mask = torch.from_numpy(tmpl.mask_bits.view(np.int64)).to(dev)
lib = _lib.load()


def run(rows, impl):
    M = B * rows
    qkv = torch.randn(M, 3 * H, device=dev).bfloat16()
    out = torch.empty(M, H, device=dev, dtype=torch.bfloat16)
    row_off = torch.tensor([b * rows for b in range(B + 1)], dtype=torch.int32, device=dev)
    row_node = torch.tensor([i for _ in range(B) for i in range(rows)], dtype=torch.int32, device=dev)
    wsb = lib.propd_attn_workspace_bytes(M, A, dh, 0)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream().cuda_stream

    def launch():
        call("propd_tree_attention", _lib.BF16, impl, B, M, A, dh, Lmax, B, max(rows, args.cap), L + n, ptr(qkv), 3 * H, ptr(kc),
             ptr(vc), ptr(slots), ptr(lens), ptr(row_off), ptr(row_node), ptr(mask), n, tmpl.words, ptr(out), H,
             ptr(ws), wsb, torch.cuda.current_stream().cuda_stream)

    launch()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        launch()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        for _ in range(args.reps):
            launch()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / args.reps
    nbytes = B * A * (2 * (L + n) * dh * 2) + 2 * M * H * 2
    print(f"B={B} kv={L} rows={rows} impl={impl}: {us:8.1f} us/launch, {nbytes / us / 1e3:7.0f} GB/s "
          f"({nbytes / us / 1e3 / 6549.4:.3f} of 6549 GB/s)")
    del st


run(args.rows, args.impl)
run(1, 0)
