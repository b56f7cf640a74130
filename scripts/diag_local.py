"""Diagnostic: in-process world (every rank on one GPU) over the SUMMA and
1.5D strategies, with CUDA-graph epochs on and off, repeated."""
import os, sys, time, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_03300_b200 as cg

cases = [("2d", 4, 1, 0, False), ("2d", 4, 1, 3, False), ("3d", 8, 1, 0, False), ("1.5d", 8, 2, 0, False),
         ("2d", 4, 1, 0, True), ("3d", 8, 1, 0, True)]
reps = int(os.environ.get("REPS", "3"))
for graph in (False, True):
    for kind, P, c, b, res in cases:
        ok = 0
        msgs = []
        for r in range(reps):
            model = cg.init_glorot([8, 6, 4], 14, 0.5)
            strat = cg.Strategy(kind, P, c, b, resident_sparse=res, graph=graph)
            t0 = time.time()
            try:
                cg.run_distributed(lambda dev: cg.generate_dataset(18, 4.0, 8, 4, 11, 12, 13, device=dev),
                                   model, strat, 3, comm="local")
                ok += 1
            except Exception as e:
                msgs.append(str(e)[:160])
        print(f"graph={graph} {kind} P={P} c={c} b={b} resident={res}: {ok}/{reps} ok", msgs[:1], flush=True)
