import sys, os, time
sys.path.insert(0, "/root/repo")
import paper_2005_03300_b200 as cg
import torch
N, E = 14249639, 230788269
DIMS = [300, 16, 16, 24]
d = cg.generate_dataset(N, E / N, DIMS[0], DIMS[-1], 1, 2, 3, device=0, generator="skip")
print("dataset", torch.cuda.mem_get_info(), flush=True)
model = cg.init_glorot(DIMS, 4, 0.5)
kind, P, repl = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
try:
    out = cg.run_distributed(d, model, cg.Strategy(kind, P, repl, reassociate=True), 2, comm="local")
    print("ok", out.losses)
except Exception as e:
    print("fail", e)
