"""Run one tree-attention case through impl=2 (tcgen05) and impl=1 (CUDA
core) and print the max error of each against a torch fp32 reference.
  python scripts/debug_tc.py B A L n [rows]     (n: grid-tree size selector)
  python scripts/debug_tc.py all                 (loop over cases in subprocesses)
"""
import ctypes
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if sys.argv[1] == "all":
    cases = [tuple(c.split(",")) for c in sys.argv[2:]] or [
        (1, 1, 1, 1), (1, 1, 100, 1), (1, 1, 128, 4), (1, 1, 300, 12), (1, 2, 1000, 12), (2, 4, 512, 12),
        (3, 4, 77, 39), (1, 32, 1024, 37), (2, 2, 4096, 160), (4, 32, 2048, 64)]
    for c in cases:
        try:
            extra = [c[4] if len(c) > 4 else None]
            r = subprocess.run([sys.executable, __file__, *map(str, c[:4]), *([str(c[4])] if len(c) > 4 else [])],
                               capture_output=True, text=True, timeout=120)
            lines = (r.stdout + r.stderr).strip().splitlines()
            print(c, "rc", r.returncode, [ln for ln in lines if "propd attn_tc" in ln][:3], lines[-3:])
        except subprocess.TimeoutExpired:
            print(c, "TIMEOUT")
    sys.exit(0)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2402_13485_b200 import _lib  # noqa: E402
from paper_2402_13485_b200._lib import call, ptr  # noqa: E402
from paper_2402_13485_b200.tree import TreeTemplate  # noqa: E402
from oracle import treedecode_port as op  # noqa: E402

B, A, L, nsel = map(int, sys.argv[1:5])
REV = os.environ.get("REV_SLOTS") == "1"
IMPLS = tuple(int(x) for x in os.environ.get("IMPLS", "1,2").split(","))
dev = torch.device("cuda:0")
paths = op.complete_tree_paths(4, 4)
paths = sorted(paths, key=lambda p: (len(p), p))[:nsel]
tmpl = TreeTemplate.from_paths(paths)
n = len(tmpl)
dh = 128
H = A * dh
lens = [max(1, L - 37 * b) for b in range(B)] if len(sys.argv) < 6 else list(map(int, sys.argv[5].split("/")))
B = len(lens)
Lmax = max(lens) + n + 8
torch.manual_seed(0)
kc = torch.randn(B, A, Lmax, dh, device=dev).bfloat16()
vc = torch.randn(B, A, Lmax, dh, device=dev).bfloat16()
M = B * n
qkv = torch.randn(M, 3 * H, device=dev).bfloat16()
keep = []


def t32(a):
    t = torch.tensor(np.asarray(a, dtype=np.int32), device=dev)
    keep.append(t)
    return t


slot_list = list(range(B))[::-1] if REV else list(range(B))
slots = t32(slot_list)
sl = [0] * B
for b, s_ in enumerate(slot_list):
    sl[s_] = lens[b]
seq_len = t32(sl)
row_off = t32([b * n for b in range(B + 1)])
row_node = t32([i for b in range(B) for i in range(n)])
mask = torch.from_numpy(tmpl.mask_bits.view(np.int64)).to(dev)
ws_bytes = _lib.load().propd_attn_workspace_bytes(M, A, dh, 0)
ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
outs = {}
for impl in IMPLS:
    out = torch.zeros(M, H, device=dev, dtype=torch.bfloat16)
    call("propd_tree_attention", _lib.BF16, impl, B, M, A, dh, Lmax, B, n, max(lens) + n, ptr(qkv), 3 * H, ptr(kc),
         ptr(vc), ptr(slots), ptr(seq_len), ptr(row_off), ptr(row_node), ptr(mask), n, tmpl.words, ptr(out), H,
         ptr(ws), ws_bytes, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    outs[impl] = out.float()
mb = tmpl.mask()
ref = torch.zeros(M, H, device=dev)
for b in range(B):
    for i in range(n):
        keys = np.concatenate([np.arange(lens[b]), lens[b] + np.flatnonzero(mb[i])])
        kk = torch.from_numpy(keys).to(dev)
        for a in range(A):
            K = kc[slot_list[b], a, kk].float()
            V = vc[slot_list[b], a, kk].float()
            s = K @ qkv[b * n + i, a * dh:(a + 1) * dh].float() / np.sqrt(dh)
            ref[b * n + i, a * dh:(a + 1) * dh] = torch.softmax(s, 0) @ V
for impl in IMPLS:
    e = (outs[impl] - ref).abs()
    print(f"impl {impl}: max err {e.max().item():.3e}  rows with err>0.05: "
          f"{sorted(set((e > 0.05).nonzero()[:, 0].tolist()))[:10]}")
if os.environ.get("TRACE") == "1":
    tb = torch.zeros(16, dtype=torch.int64, device=dev)
    lib = _lib.load()
    lib.propd_debug_trace.argtypes = [ctypes.c_void_p]
    lib.propd_debug_trace(tb.data_ptr())
    out = torch.zeros(M, H, device=dev, dtype=torch.bfloat16)
    for impl in IMPLS[::-1]:
        args = (_lib.BF16, impl, B, M, A, dh, Lmax, B, n, max(lens) + n, ptr(qkv), 3 * H, ptr(kc),
                ptr(vc), ptr(slots), ptr(seq_len), ptr(row_off), ptr(row_node), ptr(mask), n, tmpl.words, ptr(out), H,
                ptr(ws), ws_bytes, torch.cuda.current_stream().cuda_stream)
        call("propd_tree_attention", *args)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(20):
                call("propd_tree_attention", *args[:-1], torch.cuda.current_stream().cuda_stream)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 20
        byts = sum(2 * (lens[b] + n) * H * 2 for b in range(B)) + 2 * M * H * 2
        t = tb.cpu().numpy()
        print(f"impl {impl}: {us:.1f} us/launch (graph, 20 back-to-back), {byts / us / 1e3:.0f} GB/s algorithmic; "
              f"CTA(0,0,0) phases ns: {[int(x - t[0]) if x else None for x in t[:10]]}")

if os.environ.get("TRACE2") == "1":
    tb = torch.zeros(128, dtype=torch.int64, device=dev)
    lib = _lib.load()
    lib.propd_debug_trace2.argtypes = [ctypes.c_void_p]
    lib.propd_debug_trace2(tb.data_ptr())
    out = torch.zeros(M, H, device=dev, dtype=torch.bfloat16)
    for rep in range(3):
        call("propd_tree_attention", _lib.BF16, 4, B, M, A, dh, Lmax, B, n, max(lens) + n, ptr(qkv), 3 * H, ptr(kc),
             ptr(vc), ptr(slots), ptr(seq_len), ptr(row_off), ptr(row_node), ptr(mask), n, tmpl.words, ptr(out), H,
             ptr(ws), ws_bytes, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    t = tb.cpu().numpy().astype(np.int64)
    t0 = t[0]
    rel = lambda x: int(x - t0) if x else -1
    print("setup done", rel(t[1]))
    for j in range(20):
        print(f"blk {j:2d}: tma {rel(t[2+j]):7d}  S {rel(t[26+j]):7d}  sm_start {rel(t[50+j]):7d}  P {rel(t[74+j]):7d}  PV {rel(t[98+j]):7d}")
