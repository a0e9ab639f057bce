"""Time the weight-streaming GEMM vs torch.mm for the 7B projection shapes (development aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_13485_b200 import _lib  # noqa: E402
from paper_2402_13485_b200._lib import call  # noqa: E402

H = 4096
shapes = [("qkv", 3 * H, H, 1), ("wo", H, H, 1), ("w1", 4 * H, H, 1), ("w2", H, 4 * H, 1), ("lm", 32000, H, 0)]
st = torch.cuda.current_stream().cuda_stream


def bench(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


for M in tuple(int(m) for m in os.environ.get("ROWS", "1,16,48").split(",")):
    for name, N, K, acc in shapes:
        X = torch.randn(M, K, device="cuda").bfloat16()
        W = torch.randn(K, N, device="cuda").bfloat16()
        Y = torch.zeros(M, N, device="cuda")
        max_split = int(os.environ.get("MAX_SPLIT", "0"))
        t_ws = bench(lambda: call("propd_gemm_ws", M, None, N, K, X.data_ptr(), K, W.data_ptr(), N, Y.data_ptr(), N, acc,
                                  max_split, torch.cuda.current_stream().cuda_stream))
        t_mm = bench(lambda: torch.mm(X, W))
        gb = K * N * 2 / 1e9
        print(f"M={M:3d} {name:4s} N={N:6d} K={K:6d}: ws {t_ws:7.1f} us ({gb / t_ws * 1e6:6.0f} GB/s)  "
              f"torch.mm {t_mm:7.1f} us ({gb / t_mm * 1e6:6.0f} GB/s)")
