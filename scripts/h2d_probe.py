"""H2D bandwidth of a 562 MB pinned buffer (Reddit's feature tile): one copy vs the
same bytes split over 2 / 4 streams (copy engines)."""
import time
import torch

n = 561911580 // 4
src = torch.empty(n, dtype=torch.float32, pin_memory=True)
src.fill_(1.0)
dst = torch.empty(n, dtype=torch.float32, device="cuda")
for parts in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(parts)]
    chunk = (n + parts - 1) // parts
    for rep in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                dst[i * chunk:(i + 1) * chunk].copy_(src[i * chunk:(i + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"{parts} stream(s): {dt * 1e3:.2f} ms  {n * 4 / dt / 1e9:.1f} GB/s")
