"""Packed-stream check on the Amazon-shaped graph: run_distributed 1D P=1 (and 2D P=4
in-process) with CAGNET_SPMM_PACK as set in the environment; dump outputs to npz."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2005_03300_b200 as cg
N, E = 14249639, 230788269
DIMS = [300, 16, 16, 24]
tag, kind, P = sys.argv[1], sys.argv[2], int(sys.argv[3])
graph = not (len(sys.argv) > 4 and sys.argv[4] == "nograph")
E = int(sys.argv[5]) if len(sys.argv) > 5 else 2
d = cg.generate_dataset(N, E / N, DIMS[0], DIMS[-1], 1, 2, 3, device=0, generator="skip")
model = cg.init_glorot(DIMS, 4, 0.5)
out = cg.run_distributed(d, model, cg.Strategy(kind, P, 1, reassociate=True, graph=graph), E, comm="local")
arrs = {"losses": np.array(out.losses), "h_final": out.h_final}
for l in range(len(DIMS) - 1):
    arrs[f"y{l}"] = out.y_final[l]; arrs[f"w{l}"] = out.model.weights[l]; arrs[f"g{l}"] = out.g_final[l]
np.savez(f"/tmp/pack_{tag}.npz", **arrs)
print(tag, "done", repr(np.array(out.losses)))
