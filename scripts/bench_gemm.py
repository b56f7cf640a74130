"""Times cagnet_gemm_f32 shapes with CUDA events (development tool)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_03300_b200 as cg  # noqa: E402

torch.cuda.init()
s = torch.cuda.current_stream()
sp = C.c_void_p(s.cuda_stream)


def run(m, n, k, ta=0, tb=0, reps=20):
    a = torch.randn((k, m) if ta else (m, k), device="cuda")
    b = torch.randn((n, k) if tb else (k, n), device="cuda")
    c = torch.zeros((m, n), device="cuda")
    lda, ldb = a.shape[1], b.shape[1]
    f = lambda: cg.check(cg.lib.cagnet_gemm_f32(ta, tb, m, n, k, a.data_ptr(), lda, b.data_ptr(), ldb,
                                                c.data_ptr(), n, 0, 0, None, 0, None, 0, sp))
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        f()
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    byts = 4 * (m * k + k * n + m * n)
    print(f"m={m:7d} n={n:3d} k={k:6d} ta={ta} tb={tb}  {ms:8.4f} ms  {byts / ms / 1e6:8.1f} GB/s "
          f" {2 * m * n * k / ms / 1e9:8.1f} TFLOP/s", flush=True)


for n in (16, 32, 48, 64):
    run(232965, n, 600)
run(232965, 16, 604)
run(232965, 16, 16)
run(232965, 41, 16)
run(232965, 16, 41, 0, 1)
run(600, 16, 232965, 1, 0)
run(16, 16, 232965, 1, 0)
run(16, 41, 232965, 1, 0)
