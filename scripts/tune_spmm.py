#!/usr/bin/env python3
"""Times cagnet_spmm_csr_f32 on the Reddit-shaped graph (adj_t, f from argv)
for the variant in CAGNET_SPMM_TUNE.  Tuning aid, not product code."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_03300_b200 as cg  # noqa: E402
from paper_2005_03300_b200._lib import check, lib  # noqa: E402

fs = [int(x) for x in sys.argv[1:]] or [16]
n, e = 232965, 114848857
data = cg.generate_dataset(n, e / n, 16, 4, 1, 2, 3, device=0)
a = data.adj_t
rp, ci, v = a.device_ptrs()
s = torch.cuda.current_stream().cuda_stream
for f in fs:
    ld = (f + 3) // 4 * 4
    H = torch.rand(n, ld, device="cuda")
    T = torch.zeros(n, ld, device="cuda")
    ref = None

    def run():
        check(lib.cagnet_spmm_csr_f32(a.n_rows, a.n_cols, a.nnz, rp, ci, v, H.data_ptr(), ld, f,
                                      T.data_ptr(), ld, 0, s))
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for _ in range(10):
        flush.zero_()
        st.record()
        run()
        en.record()
        torch.cuda.synchronize()
        ts.append(st.elapsed_time(en))
    ts.sort()
    st.record()
    for _ in range(10):
        run()
    en.record()
    torch.cuda.synchronize()
    b2b = st.elapsed_time(en) / 10
    print(f"variant={os.environ.get('CAGNET_SPMM_TUNE', '0')} f={f} flushed median {ts[5]:.4f} ms "
          f"back-to-back {b2b:.4f} ms  checksum {float(T[:, :f].double().sum()):.6e}", flush=True)
