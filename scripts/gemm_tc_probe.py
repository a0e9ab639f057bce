"""Many-row projection throughput: propd_gemm (tcgen05, 128 x 256 tiles, the
layer's epilogue: fp32 residual add (split-K at few tiles) for W_o / W_2, bf16
/ fp32 stores otherwise) vs torch.mm (cuBLAS, bf16 out) on the 7B layer shapes,
TFLOP/s from CUDA events over 20 back-to-back launches.

  python scripts/gemm_tc_probe.py [--rows 256,512,1024,2048,4096]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_13485_b200 import _lib  # noqa: E402
from paper_2402_13485_b200._lib import call, ptr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rows", default="256,512,1024,2048,4096")
ap.add_argument("--reps", type=int, default=20)
args = ap.parse_args()
_lib.load()
dev = torch.device("cuda")
st = torch.cuda.current_stream().cuda_stream
shapes = [("QKV", 4096, 12288), ("W_o", 4096, 4096), ("W_1", 4096, 16384), ("W_2", 16384, 4096), ("LM", 4096, 32000)]
for M in map(int, args.rows.split(",")):
    for name, K, N in shapes:
        X = torch.randn(M, K, device=dev).bfloat16()
        W = (torch.randn(K, N, device=dev) / K ** 0.5).bfloat16()
        # the layer's epilogue: residual add for W_o / W_2 (fp32 Y), bf16 / fp32 stores otherwise
        add = name in ("W_o", "W_2")
        Y = torch.zeros(M, N, device=dev, dtype=torch.float32 if (add or name == "LM") else torch.bfloat16)
        mode = _lib.EPI_ADD_F32 if add else (_lib.EPI_STORE_F32 if name == "LM" else _lib.EPI_STORE)
        epi = _lib.GemmEpi(mode=mode, Y=ptr(Y), ldy=N)
        Yc = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        f = lambda: call("propd_gemm", _lib.BF16, M, None, N, K, ptr(X), K, ptr(W), N, epi, st)
        g = lambda: torch.mm(X, W, out=Yc)
        res = {}
        for lab, fn in (("propd", f), ("cublas", g)):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / args.reps * 1e3
            res[lab] = (us, 2 * M * N * K / (us * 1e-6) / 1e12)
        print(f"M={M:5d} {name:4s} N={N:6d} K={K:6d}  propd {res['propd'][0]:8.1f} us {res['propd'][1]:7.1f} TF/s   "
              f"cublas {res['cublas'][0]:8.1f} us {res['cublas'][1]:7.1f} TF/s   ratio {res['cublas'][0] / res['propd'][0]:.2f}",
              flush=True)
