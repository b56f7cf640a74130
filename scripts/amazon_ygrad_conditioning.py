"""Amazon-shaped weight gradients (14.2 M-row reductions) of a 1D single-rank
run against fp64 recomputations on the GPU from the run's own activations:
Y0 = H0^T (A G1), Y1 = H1^T (A G2), Y2 = (A^T H2)^T G3 (narrow-first widening
layer).  CAGNET_HTS_CHUNK_ROWS bounds the tensor-core split length."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_03300_b200 as cg

N, E = 14249639, 230788269
DIMS = [300, 16, 16, 24]
d = cg.generate_dataset(N, E / N, DIMS[0], DIMS[-1], 1, 2, 3, device=0, generator="skip")
model = cg.init_glorot(DIMS, 4, 0.5)
t = cg.make_trainer(d, model, cg.Strategy("1d", 1, reassociate=True))
t.distribute()
t.run_epochs(2)
gpu = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.float64)).cuda()
ys = [t.y(l).astype(np.float64) for l in range(3)]
H = [gpu(t.h_tile(l)) for l in range(3)]
G = [gpu(t.g_tile(l)) for l in range(3)]
del t
rp, ci, v = d.csr(0).download()
A = torch.sparse_csr_tensor(torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda(),
                            torch.from_numpy(v.astype(np.float64)).cuda(), size=(N, N))
rp, ci, v = d.csr(1).download()
At = torch.sparse_csr_tensor(torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda(),
                             torch.from_numpy(v.astype(np.float64)).cuda(), size=(N, N))
truth = [(H[0].T @ (A @ G[0])).cpu().numpy(), (H[1].T @ (A @ G[1])).cpu().numpy(),
         ((At @ H[2]).T @ G[2]).cpu().numpy()]
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
tag = os.environ.get("CAGNET_HTS_CHUNK_ROWS", "8192 (default)")
print(f"chunk={tag}: " + ", ".join(f"Y{l} vs fp64 {rel(ys[l], truth[l]):.2e}" for l in range(3)))
