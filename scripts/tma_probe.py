"""TMA streaming ceiling probe (development aid)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_13485_b200 import _lib  # noqa: E402

lib = _lib.load()
lib.propd_debug_tma_stream.argtypes = [ctypes.c_void_p] * 2 + [ctypes.c_int] * 5 + [ctypes.c_void_p]
B, A, L = 64, 32, 4096
Lmax = L + 64
kc = torch.zeros(B, A, Lmax, 128, device="cuda", dtype=torch.bfloat16)
vc = torch.zeros_like(kc)
st = torch.cuda.current_stream().cuda_stream
for grid in (148, 296):
    for _ in range(2):
        rc = lib.propd_debug_tma_stream(kc.data_ptr(), vc.data_ptr(), B, A, Lmax, L // 64, grid, st)
        assert rc == 0, lib.propd_last_error()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        lib.propd_debug_tma_stream(kc.data_ptr(), vc.data_ptr(), B, A, Lmax, L // 64, grid, st)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 5
    byts = B * A * L * 128 * 2 * 2
    print(f"grid {grid}: {us:.1f} us, {byts / us / 1e3:.0f} GB/s (TMA 64x64 boxes, 6-stage ring, no compute)")
x = torch.empty(B * A * L * 128 * 2, dtype=torch.bfloat16, device="cuda")
for _ in range(2):
    x.sum()
e0.record()
for _ in range(5):
    x.float().sum() if False else torch.sum(x)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / 5
print(f"torch.sum read of the same bytes: {us:.1f} us, {x.numel() * 2 / us / 1e3:.0f} GB/s")
