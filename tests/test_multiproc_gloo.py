"""N > 1 host-side path on CPU: world_size-2 gloo processes run the
launcher's bootstrap (rank 0 makes the NCCL unique id, the group broadcasts
it) and each rank derives its partition geometry through the C-ABI; the
gathered tiles must partition every embedding matrix exactly once
(test_dist.cpp:167-198) for all four strategies."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, results):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2005_03300_b200 as cg

    buf = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        buf.copy_(torch.frombuffer(bytearray(cg.comm_unique_id()), dtype=torch.uint8))
    dist.broadcast(buf, 0)
    ids = [torch.zeros(128, dtype=torch.uint8) for _ in range(world)]
    dist.all_gather(ids, buf)
    same_id = all(bool(torch.equal(ids[0], x)) for x in ids)

    n, width = 13, 6
    report = {}
    for kind, P, c in (("1d", 2, 1), ("1.5d", 8, 2), ("2d", 4, 1), ("3d", 8, 1)):
        grid = cg.ProcessGrid(cg.Strategy(kind, P, c))
        # Ranks of the strategy are dealt round-robin over the processes.
        mine = [list(grid.tile(n, r, width)) + [r] for r in range(rank, P, world)]
        t = torch.tensor(mine + [[-1] * 6] * (P - len(mine)), dtype=torch.int64)
        gathered = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(gathered, t)
        report[kind] = [row for g in gathered for row in g.tolist() if row[0] >= 0]
    if rank == 0:
        results.put((same_id, report))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_bootstrap_and_geometry():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    same_id, report = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert same_id
    n, width = 13, 6
    for kind, rows in report.items():
        cover = np.zeros((n, width), np.int64)
        seen = set()
        for r0, r1, c0, c1, owner, rank in rows:
            seen.add(rank)
            if owner == rank:
                cover[r0:r1, c0:c1] += 1
        assert np.all(cover == 1), kind
        assert seen == set(range(len(rows))), kind
