"""Times the C-ABI SpMM at several widths f on a random 116K x 116K tile (247 nnz/row),
the shape of a 2D P=4 Reddit tile.  Not a test; a tuning aid."""
import ctypes, sys, os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_03300_b200 as cg
from paper_2005_03300_b200 import _lib
L = _lib.lib
n, deg = 116483, 247
g = torch.Generator(device="cuda").manual_seed(1)
cols = torch.randint(0, n, (n * deg,), device="cuda", generator=g, dtype=torch.int32).view(n, deg).sort(dim=1).values.reshape(-1).contiguous()
rp = (torch.arange(n + 1, device="cuda", dtype=torch.int64) * deg).contiguous()
vals = torch.rand(n * deg, device="cuda", generator=g)
for f in [8, 16, 20, 21, 24, 32, 41, 44]:
    ld = (f + 3) // 4 * 4
    H = torch.zeros(n, ld, device="cuda"); H[:, :f] = torch.rand(n, f, device="cuda", generator=g)
    T = torch.zeros(n, ld, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    def run():
        rc = L.cagnet_spmm_csr_f32(n, n, n * deg, rp.data_ptr(), cols.data_ptr(), vals.data_ptr(), H.data_ptr(), ld, f,
                                   T.data_ptr(), ld, 0, ctypes.c_void_p(s))
        assert rc == 0
    for _ in range(3): run()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): run()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    print(f"f={f:3d} ld={ld:3d}  {ms:.4f} ms  gathered {n*deg*f*4/ms/1e9:.0f} GB/s", flush=True)
