"""Repeat a multi-rank in-process run and compare with the 1D P=1 outcome (race hunt)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2005_03300_b200 as cg
cfg = sys.argv[1]
if cfg == "amazon":
    N, E, DIMS, gen = 14249639, 230788269, [300, 16, 16, 24], "skip"
else:
    N, E, DIMS, gen = 232965, 114848857, [602, 16, 16, 41], "reference"
kind, P = sys.argv[2], int(sys.argv[3])
reps = int(sys.argv[4])
opts = dict(a.split("=") for a in sys.argv[5:])
d = cg.generate_dataset(N, E / N, DIMS[0], DIMS[-1], 1, 2, 3, device=0, generator=gen)
model = cg.init_glorot(DIMS, 4, 0.5)
epochs = int(opts.pop("epochs", 2))
skw = {k: (v == "1") if k in ("graph", "resident_sparse", "reassociate") else int(v) for k, v in opts.items()}
skw.setdefault("reassociate", True)
base = cg.run_distributed(d, model, cg.Strategy("1d", 1, reassociate=skw["reassociate"], graph=skw.get("graph", True)), epochs)
def rel(a, b): return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
bad = 0
for r in range(reps):
    t = time.time()
    out = cg.run_distributed(d, model, cg.Strategy(kind, P, 2 if kind == "1.5d" else 1, **skw), epochs, comm="local")
    errs = {f"y{l}": rel(out.y_final[l], base.y_final[l]) for l in range(len(DIMS) - 1)}
    errs["h"] = rel(out.h_final, base.h_final)
    worst = max(errs.values())
    bad += worst > 1e-4
    print(f"rep {r} {time.time()-t:.1f}s worst {worst:.2e}", {k: f"{v:.1e}" for k, v in errs.items()}, flush=True)
print(f"{cfg} {kind} P={P} {opts} epochs={epochs}: {bad}/{reps} bad")
