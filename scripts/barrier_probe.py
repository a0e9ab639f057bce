"""Cost of a grid barrier among 288 co-resident CTAs (development aid):
impl 0 = single-counter atomic arrive + departure re-arm, impl 1 = spread
fire-and-forget arrivals over 16 counters, warp-polled sum."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_13485_b200 import _lib  # noqa: E402

lib = _lib.load()
bar = torch.zeros(128, device="cuda", dtype=torch.int32)
for impl in (0, 1):
    for ctas in (148, 288):
        for iters in (1, 101):
            st = torch.cuda.current_stream().cuda_stream
            lib.propd_debug_barrier_bench(ctas, iters, ctypes.c_void_p(bar.data_ptr()), impl, ctypes.c_void_p(st))
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            lib.propd_debug_barrier_bench(ctas, iters, ctypes.c_void_p(bar.data_ptr()), impl, ctypes.c_void_p(st))
            e1.record()
            torch.cuda.synchronize()
            print(f"impl {impl} ctas {ctas} iters {iters}: {e0.elapsed_time(e1) * 1e3:8.1f} us")
