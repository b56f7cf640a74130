"""Device timeline of graph-replayed epochs (CUPTI via torch.profiler), one file per rank.
Analysis aid only (numbers under a profiler are never bench values).
  torchrun --nproc-per-node N scripts/timeline.py --gpus N [--strategy 1d] [--config reddit]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import torch


def main():
    args = bench.parse()
    cfg = bench.CONFIGS[args.config]
    import paper_2005_03300_b200 as cg
    rank, world, local = bench.dist_env()
    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist
    repl = args.repl or (2 if args.strategy == "1.5d" else 1)
    strat = cg.Strategy(args.strategy, world, repl, args.block, reassociate=not args.reference_order,
                        fuse=args.fuse, overlap=args.overlap)
    nid = None
    if world > 1:
        buf = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            buf.copy_(torch.frombuffer(bytearray(cg.comm_unique_id()), dtype=torch.uint8))
        pg.broadcast(buf, 0)
        nid = bytes(buf.cpu().numpy().tobytes())
    data = cg.generate_dataset(cfg["n"], cfg["degree"], cfg["dims"][0], cfg["dims"][-1],
                               device=local, generator=cfg["generator"], **bench.SEEDS)
    model = cg.init_glorot(cfg["dims"], bench.SEED_W, bench.LR)
    tr = cg.make_trainer(data, model, strat, rank, nid)
    tr.distribute()
    tr.run_epochs(3)
    torch.cuda.synchronize()
    if pg:
        pg.barrier()
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            tr.epoch_async()
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    ev.sort(key=lambda e: e.time_range.start)
    t0 = ev[0].time_range.start if ev else 0
    out = [(round(e.time_range.start - t0, 1), round(e.time_range.end - e.time_range.start, 1), e.name[:90])
           for e in ev]
    os.makedirs("gpurun_out", exist_ok=True)
    with open(f"gpurun_out/timeline_{args.strategy}_n{world}_r{rank}.txt", "w") as f:
        for s, d, n in out:
            f.write(f"{s:10.1f} {d:8.1f}  {n}\n")
    if pg:
        pg.barrier()


if __name__ == "__main__":
    main()
