import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2005_03300_b200 as cg
n, e = 232965, 114848857
data = cg.generate_dataset(n, e / n, 16, 4, 1, 2, 3, device=0)
rp, ci, v = data.adj_t.download()
rp.astype(np.int64).tofile("/tmp/csr_rp.bin"); ci.astype(np.int32).tofile("/tmp/csr_ci.bin"); v.astype(np.float32).tofile("/tmp/csr_v.bin")
print("dumped", rp[-1])
