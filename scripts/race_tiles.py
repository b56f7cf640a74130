"""Race hunt: P in-process ranks (Python threads over the C-ABI), epoch by epoch;
every rank's h / g / y tiles snapshotted after each epoch and compared across reps."""
import os, sys, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2005_03300_b200 as cg
kind, P, reps, E = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
N, EE, DIMS = 232965, 114848857, [602, 16, 16, 41]
L = len(DIMS) - 1
datas = [cg.generate_dataset(N, EE / N, DIMS[0], DIMS[-1], 1, 2, 3, device=0) for _ in range(P)]
model = cg.init_glorot(DIMS, 4, 0.5)
strat = cg.Strategy(kind, P, 1, reassociate=True, graph=False)

def par(fn):
    errs = []
    def body(r):
        try: fn(r)
        except Exception as e:
            errs.append(e); cg.comm_local_abort(nid, str(e))
    th = [threading.Thread(target=body, args=(r,)) for r in range(P)]
    [x.start() for x in th]; [x.join() for x in th]
    assert not errs, errs

b = cg.Trainer(datas[0], model, cg.Strategy("1d", 1, reassociate=True, graph=False), 0, None)
b.distribute()
base = []
for e in range(E):
    b.run_epochs(1)
    base.append({f"y{l}": b.y(l) for l in range(L)} | {f"w{l}": b.weight(l) for l in range(L)})
del b
def rel(a, c): return float(np.linalg.norm(a - c) / max(np.linalg.norm(c), 1e-300))
snaps = []
for rep in range(reps):
    nid = cg.comm_local_id(P, 0)
    tr = [None] * P
    def mk(r):
        t = cg.Trainer(datas[r], model, strat, r, nid); t.distribute(); tr[r] = t
    par(mk)
    per_epoch = []
    for e in range(E):
        par(lambda r: tr[r].run_epochs(1))
        s = {}
        for r in range(P):
            t = tr[r]
            for l in range(L + 1):
                s[f"r{r}_h{l}"] = t.h_tile(l)
            for l in range(L):
                s[f"r{r}_g{l}"] = t.g_tile(l); s[f"r{r}_y{l}"] = t.y(l); s[f"r{r}_w{l}"] = t.weight(l)
        per_epoch.append(s)
    snaps.append(per_epoch)
    for t in tr: t.free() if hasattr(t, "free") else None
    del tr
    print("rep", rep, "vs 1D:", [{k: f"{rel(per_epoch[e]['r0_' + k], base[e][k]):.1e}" for k in base[e]} for e in range(E)], flush=True)

for rep in range(1, reps):
    for e in range(E):
        a, b = snaps[0][e], snaps[rep][e]
        diffs = {k: float(np.max(np.abs(a[k] - b[k]))) for k in a if a[k].shape == b[k].shape}
        bad = {k: f"{v:.1e}" for k, v in diffs.items() if v > 0}
        print(f"rep {rep} epoch {e}: {len(bad)} differing arrays", dict(sorted(bad.items())[:40]), flush=True)
