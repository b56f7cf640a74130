"""Multi-GPU e2e diagnosis (torchrun): per-rank wall time of each phase of the
pipelined host-buffer loop (prefetch_host, step_prefetched) and of step_host."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist
import paper_2005_03300_b200 as cg
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", init_method="env://", device_id=torch.device("cuda", local))
p2p = os.environ.get("P2P", "1") == "1"
N, E, DIMS = 232965, 114848857, [602, 16, 16, 41]
data = cg.generate_dataset(N, E / N, DIMS[0], DIMS[-1], 1, 2, 3, device=local)
model = cg.init_glorot(DIMS, 4, 0.5)
nid = cg.comm_unique_id() if rank == 0 else bytes(128)
obj = [nid]; dist.broadcast_object_list(obj, src=0); nid = obj[0]
t = cg.make_trainer(data, model, cg.Strategy("1d", world, reassociate=True, p2p=p2p), rank, nid)
t.distribute()
r0, r1, c0, c1, _ = t.tile(rank, DIMS[0])
feats = data.features()[r0:r1, c0:c1]
x = torch.empty(feats.shape, dtype=torch.float32, pin_memory=True); x.numpy()[:] = feats
lab = torch.empty(r1 - r0, dtype=torch.int32, pin_memory=True); lab.numpy()[:] = data.labels()[r0:r1]
for _ in range(3): t.step_host(x.numpy(), lab.numpy())
dist.barrier()
K = 10
sh = []
for _ in range(K):
    a = time.perf_counter(); t.step_host(x.numpy(), lab.numpy()); sh.append((time.perf_counter() - a) * 1e3)
dist.barrier()
pf, st = [], []
a0 = time.perf_counter()
a = time.perf_counter(); t.prefetch_host(x.numpy(), lab.numpy()); pf.append((time.perf_counter() - a) * 1e3)
for k in range(K):
    if k + 1 < K:
        a = time.perf_counter(); t.prefetch_host(x.numpy(), lab.numpy()); pf.append((time.perf_counter() - a) * 1e3)
    a = time.perf_counter(); t.step_prefetched(); st.append((time.perf_counter() - a) * 1e3)
tot = (time.perf_counter() - a0) * 1e3 / K
print(f"rank {rank} p2p={p2p} step_host med {statistics.median(sh):.2f} | pipelined {tot:.2f}/step: "
      f"prefetch {[round(v,2) for v in pf[:5]]} step {[round(v,2) for v in st[:5]]}", flush=True)
dist.barrier()
dist.destroy_process_group()
