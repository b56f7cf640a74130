"""NCCL collective timing on this box (torch.distributed, same NCCL): the
ceiling for the 1D panel all-gather (n x 16 fp32 = 15 MB) and small
all-reduces.  Run with torchrun.  Tuning aid."""
import os
import torch
import torch.distributed as dist

dist.init_process_group("nccl")
r, w = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dev = torch.device("cuda")
for mb in (1, 4, 15, 60):
    n = mb * 1024 * 1024 // 4 // w * w
    out = torch.zeros(n, device=dev)
    inp = out[r * (n // w):(r + 1) * (n // w)]
    for _ in range(5):
        dist.all_gather_into_tensor(out, inp)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        dist.all_gather_into_tensor(out, inp)
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) / 20
    if r == 0:
        print(f"allgather {mb:3d} MB: {t * 1e3:8.1f} us  busbw {(w - 1) / w * n * 4 / t / 1e6:7.1f} GB/s", flush=True)
x = torch.ones(4096, device=dev)
for _ in range(5):
    dist.all_reduce(x)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(50):
    dist.all_reduce(x)
e.record()
torch.cuda.synchronize()
if r == 0:
    print(f"allreduce 16 KB: {s.elapsed_time(e) / 50 * 1e3:.1f} us", flush=True)
dist.destroy_process_group()
