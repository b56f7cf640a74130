import ctypes as C, numpy as np, sys
sys.path.insert(0, '.')
import paper_2005_03300_b200 as cg
import torch
torch.cuda.init()
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
rng = np.random.default_rng(0)
for (m, n, k, ta, tb) in [(128, 16, 32, 0, 0), (128, 16, 8, 0, 0), (256, 16, 64, 0, 0), (128, 16, 32, 1, 0), (128, 16, 32, 0, 1)]:
    a = rng.standard_normal((k, m) if ta else (m, k)).astype(np.float32)
    b = rng.standard_normal((n, k) if tb else (k, n)).astype(np.float32)
    A = torch.from_numpy(a).cuda(); B = torch.from_numpy(b).cuda(); Cm = torch.zeros((m, n), device='cuda')
    cg.check(cg.lib.cagnet_gemm_f32(ta, tb, m, n, k, A.data_ptr(), A.shape[1], B.data_ptr(), B.shape[1], Cm.data_ptr(), n, 0, 0, None, 0, None, 0, s))
    torch.cuda.synchronize()
    got = Cm.cpu().numpy()
    want = (a.T if ta else a).astype(np.float64) @ (b.T if tb else b).astype(np.float64)
    err = np.abs(got - want).max() / np.abs(want).max()
    print((m, n, k, ta, tb), 'maxrel', err, 'got[0,:4]', got[0, :4], 'want', want[0, :4], 'nonzero', np.count_nonzero(got))
    if err > 1e-3:
        # diagnose: check if got matches a permutation / transposed variant
        for name, cand in [('AtB', None)]:
            pass
