#!/usr/bin/env python3
"""SpMM column-blocking sweep on a large skip-generated graph (tuning aid):
times A^T H (f=16) as nb column-block passes (extracted CSR blocks, the last
passes accumulating) for several nb.  Usage: tune_spmm_big.py n degree nb..."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_03300_b200 as cg  # noqa: E402
from paper_2005_03300_b200._lib import check, lib  # noqa: E402

n, deg = int(sys.argv[1]), float(sys.argv[2])
nbs = [int(x) for x in sys.argv[3:]]
data = cg.generate_dataset(n, deg, 16, 4, 1, 2, 3, device=0, generator="skip")
a = data.adj_t
f = 16
H = torch.rand(n, f, device="cuda")
T = torch.zeros(n, f, device="cuda")
s = torch.cuda.current_stream().cuda_stream
print(f"n={n} nnz={a.nnz} H={n * f * 4 / 1e6:.0f} MB", flush=True)
for nb in nbs:
    step = (n + nb - 1) // nb
    blocks = [cg.extract_block(a, 0, n, b * step, min(n, (b + 1) * step)) for b in range(nb)]
    ptrs = [b.device_ptrs() for b in blocks]

    def run():
        for b, (blk, (rp, ci, v)) in enumerate(zip(blocks, ptrs)):
            c0 = b * step
            check(lib.cagnet_spmm_csr_f32(blk.n_rows, blk.n_cols, blk.nnz, rp, ci, v,
                                          H.data_ptr() + c0 * f * 4, f, f, T.data_ptr(), f,
                                          int(b > 0), s))
    run()
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st.record()
    for _ in range(3):
        run()
    en.record()
    torch.cuda.synchronize()
    print(f"nb={nb:3d} panel={step * f * 4 / 1e6:7.1f} MB  {st.elapsed_time(en) / 3:8.3f} ms", flush=True)
    del blocks
