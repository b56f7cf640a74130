import sys, numpy as np
def rel(a, b): return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
base = np.load(f"/tmp/pack_{sys.argv[1]}.npz")
for t in sys.argv[2:]:
    o = np.load(f"/tmp/pack_{t}.npz")
    print(t, "vs", sys.argv[1], {k: f"{rel(o[k], base[k]):.2e}" for k in base.files})
