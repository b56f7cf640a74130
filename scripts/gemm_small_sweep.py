"""Amazon-shaped narrow GEMMs (14.25 M rows, 16 -> 16) through cagnet_gemm_f32:
the quad kernel (rows-in-flight R) vs the row-team kernel; bytes = 4(mk + kn + mn)
(+ 4mn for the relu side output)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2005_03300_b200 as cg

m, k, n = 14249639, 16, 16
A = torch.randn(m, 16, device="cuda")
W = torch.randn(16, 16, device="cuda")
C = torch.zeros(m, 16, device="cuda")
H = torch.zeros(m, 16, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for label, epi, aux in (("H.W (relu side output)", 1, H), ("H.W", 0, None)):
    for reps in (1, 20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            cg.check(cg.lib.cagnet_gemm_f32(0, 0, m, n, k, A.data_ptr(), 16, W.data_ptr(), 16, C.data_ptr(), 16,
                                            0, epi, None, 0, aux.data_ptr() if aux is not None else None, 16, s))
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    byts = 4 * (m * k + k * n + m * n) + (4 * m * n if epi else 0)
    print(f"{os.environ.get('CAGNET_GEMM_QUAD','1')}/{os.environ.get('CAGNET_GEMM_QUAD_R','2')} {label}: "
          f"{ms:.4f} ms  {byts / ms / 1e6:.0f} GB/s")
