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


def pad4(x):
    return (x + 3) // 4 * 4


def run(m, n, k, ta=0, tb=0, reps=20, epi=0):
    a = torch.randn((k, pad4(m)) if ta else (m, pad4(k)), device="cuda")
    b = torch.randn((n, pad4(k)) if tb else (k, pad4(n)), device="cuda")
    c = torch.zeros((m, pad4(n)), device="cuda")
    aux = torch.randn((m, pad4(n)), device="cuda")
    lda, ldb, ldc = a.shape[1], b.shape[1], c.shape[1]
    f = lambda: cg.check(cg.lib.cagnet_gemm_f32(ta, tb, m, n, k, a.data_ptr(), lda, b.data_ptr(), ldb,
                                                c.data_ptr(), ldc, 0, epi, aux.data_ptr(), ldc,
                                                aux.data_ptr(), ldc, sp))
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
    print(f"m={m:7d} n={n:3d} k={k:6d} ta={ta} tb={tb} epi={epi} {ms:8.4f} ms  {byts / ms / 1e6:8.1f} GB/s "
          f" {2 * m * n * k / ms / 1e9:8.1f} TFLOP/s", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        m, n, k, ta, tb, epi = (int(x) for x in sys.argv[1:7])
        run(m, n, k, ta, tb, reps=int(os.environ.get("REPS", "20")), epi=epi)
        sys.exit(0)
    run(232965, 16, 602)
    run(232965, 16, 16)
    run(232965, 16, 16, epi=1)
    run(232965, 41, 16)
    run(232965, 16, 41, 0, 1)
    run(232965, 16, 16, 0, 1, epi=2)
    run(602, 16, 232965, 1, 0)
    run(16, 16, 232965, 1, 0)
    run(16, 41, 232965, 1, 0)
