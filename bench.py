#!/usr/bin/env python3
"""Benchmark of the B200 CAGNET full-batch GCN training step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config reddit]
                    [--strategy 1d|1.5d|2d|3d] [--repl c] [--impl ours|reference]

N > 1 is launched with torchrun (one process per GPU, NCCL over NVLink).
A step is one full-batch training epoch (forward, loss, backward, SGD) of the
GCN on the synthetic graph of BASELINE.json's config, inputs resident in HBM.
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GCN epoch time (ms) at 1/2/4/8 B200 per 1D/1.5D/2D/3D; SpMM GB/s vs HBM"
REDDIT_N, REDDIT_E = 232965, 114848857
CONFIGS = {
    # BASELINE.json configs[0]
    "config1": dict(n=4096, degree=16.0, dims=[128, 16, 8], generator="reference",
                    label="ER n=4096 d=16, 2-layer GCN {128,16,8}"),
    # configs[1]/[2]: Reddit-shaped, the bit-exact reference ER generator on the GPU
    "reddit": dict(n=REDDIT_N, degree=REDDIT_E / REDDIT_N, dims=[602, 16, 16, 41],
                   generator="reference",
                   label="Reddit-shaped ER n=232965 nnz=115M f=602, 3-layer GCN {602,16,16,41}"),
    # configs[3]: Amazon-shaped, O(nnz) ER-shaped generator
    "amazon": dict(n=14249639, degree=230788269 / 14249639, dims=[300, 16, 16, 24],
                   generator="skip",
                   label="Amazon-shaped ER n=14.2M nnz=245M f=300, 3-layer GCN {300,16,16,24}"),
    # configs[4]: Protein-shaped (BASELINE's 1.3B edges)
    "protein": dict(n=8745542, degree=1.3e9 / 8745542, dims=[128, 16, 16, 256], generator="skip",
                    label="Protein-shaped ER n=8.7M nnz=1.3B f=128, 3-layer GCN {128,16,16,256}"),
}
SEEDS = dict(seed_graph=1, seed_features=2, seed_labels=3)
SEED_W, LR = 4, 0.5


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="reddit", choices=sorted(CONFIGS))
    p.add_argument("--strategy", default="1d", choices=["1d", "1.5d", "2d", "3d"])
    p.add_argument("--repl", type=int, default=0, help="1.5D replication (default 2 when 1.5d)")
    p.add_argument("--block", type=int, default=0)
    p.add_argument("--reference-order", action="store_true",
                   help="propagate as the reference does, (A^T H) W, instead of the default "
                        "narrow-first A^T (H W) on 1D/1.5D (same product)")
    p.add_argument("--overlap", action="store_true",
                   help="1D peer-memory stages: own-block SpMM overlapped with the pushes")
    p.add_argument("--no-alt", action="store_true",
                   help="skip timing the other propagation order")
    p.add_argument("--fuse", type=int, default=1,
                   help="fused SpMM row epilogues: 0 off, 1 ReLU/relu' (default), 2 + dense W")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    """Samples SM clock and clock-event (throttle) reasons of one GPU every
    ~2 ms through NVML in a thread, so even a short timed region gets
    samples (nvidia-smi's 100 ms loop missed a 20 ms region)."""

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            visible = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(visible.split(",")[self.device]) if visible else self.device
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception:
            self._t = None
        return self

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                reasons = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.samples.append((mhz, reasons))
            except Exception:
                pass
            time.sleep(0.002)

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"],
                    "samples": 0}
        nv = self._nv
        names = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                 "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                 "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                 "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap,
                 "hw_power_brake_slowdown": nv.nvmlClocksEventReasonHwPowerBrakeSlowdown}
        seen = sorted({k for _, r in self.samples for k, bit in names.items() if r & bit})
        return {"sm_mhz": statistics.median(m for m, _ in self.samples),
                "sm_max_mhz": self.max_mhz, "reasons": seen, "samples": len(self.samples),
                "source": "NVML every ~2 ms during the timed region"}


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref = the unmodified reference sources), full size
# ---------------------------------------------------------------------------
def ref_threads() -> int:
    return max(1, min(os.cpu_count() or 1, 64))


def reference_session(cfg, ranks):
    """The reference's run_distributed (dist_common.cpp:205-222), 1D with
    `ranks` rank threads, on the config's FULL graph: the raw ER graph is the
    reference generator's (csr.cpp:195-218) output, produced on all host
    threads by the oracle's jump-ahead restatement (bit-identical, pinned in
    tests/test_oracle.py) because the reference's own loop is single-threaded
    (~8 min for Reddit); features / labels / make_dataset / distribute are
    the reference's own code.  Returns (session, setup dict)."""
    import oracle
    orc, ref = oracle.Oracle(), oracle.Ref()
    n, dims = cfg["n"], cfg["dims"]
    t0 = time.perf_counter()
    raw = orc.er_generate_mt(n, cfg["degree"], SEEDS["seed_graph"], ref_threads())
    t1 = time.perf_counter()
    x = orc.random_features(n, dims[0], SEEDS["seed_features"])
    y = orc.random_labels(n, dims[-1], SEEDS["seed_labels"])
    data = ref.dataset_make(raw, x, y, dims[-1])
    del x, raw
    t2 = time.perf_counter()
    model = ref.model(dims, SEED_W, LR)
    sess = ref.session(data, model, "1d", ranks)
    t3 = time.perf_counter()
    setup = {"er_threads_s": round(t1 - t0, 1), "make_dataset_s": round(t2 - t1, 1),
             "distribute_s": round(t3 - t2, 1), "nnz": int(data.nnz)}
    sess._keep = (data, model)
    return sess, setup


def run_reference(args, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    try:
        import oracle
        if not oracle.ref_available():
            raise FileNotFoundError("oracle/_ref/libcagnet_ref.so missing")
    except Exception as e:  # pragma: no cover
        print(json.dumps({"impl": "reference", "unavailable": str(e)}))
        return
    if cfg["generator"] != "reference":
        print(json.dumps({"impl": "reference", "unavailable":
                          "the reference's O(n^2) ER generator and fp64 dense features do not "
                          "scale to this config (SURVEY 8d); run --config reddit"}))
        return
    threads = ref_threads()
    sess, setup = reference_session(cfg, threads)
    for _ in range(args.warmup):
        sess.epoch()
    times = [sess.epoch() for _ in range(args.steps)]
    ms = statistics.mean(times) * 1e3
    desc = (f"reference run_distributed 1D P={threads} rank threads on the full graph "
            f"(n={cfg['n']}, nnz={setup['nnz']}), {args.steps} timed epochs after "
            f"{args.warmup} warm-up epochs, mean epoch wall time")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(ms, 3), "unit": "ms",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 3), "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["label"], "strategy": "1d", "ranks": threads},
        "cpu_baseline": {"value": round(ms, 3), "unit": "ms", "cores": threads,
                         "kind": "reference", "sample": desc},
        "e2e": {"value": round(ms, 3), "unit": "ms", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "epoch_ms": [round(t * 1e3, 1) for t in times],
        "setup_s": setup,
    }
    print(json.dumps(line))


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def load_traffic(kernel_name):
    """dram bytes per launch of `kernel_name` from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        return json.load(open(path)).get(kernel_name)
    except Exception:
        return None


def run_ours(args, cfg):
    import torch
    import paper_2005_03300_b200 as cg

    rank, world, local = dist_env()
    N = args.gpus
    if world != N:
        raise SystemExit(f"--gpus {N} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist
    kind = args.strategy
    repl = args.repl or (2 if kind == "1.5d" else 1)
    strat = cg.Strategy(kind, N, repl, args.block, reassociate=not args.reference_order,
                        fuse=args.fuse, overlap=args.overlap)

    # NCCL bootstrap for the library's own communicators.
    nid = None
    if world > 1:
        buf = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            buf.copy_(torch.frombuffer(bytearray(cg.comm_unique_id()), dtype=torch.uint8))
        pg.broadcast(buf, 0)
        nid = bytes(buf.cpu().numpy().tobytes())

    t0 = time.perf_counter()
    data = cg.generate_dataset(cfg["n"], cfg["degree"], cfg["dims"][0], cfg["dims"][-1],
                               device=local, generator=cfg["generator"], **SEEDS)
    gen_s = time.perf_counter() - t0
    model = cg.init_glorot(cfg["dims"], SEED_W, LR)
    trainer = cg.make_trainer(data, model, strat, rank, nid)
    trainer.distribute()
    stream = torch.cuda.ExternalStream(trainer.stream())

    def barrier():
        torch.cuda.synchronize()
        if pg:
            pg.barrier()
            torch.cuda.synchronize()

    # warm-up (untimed)
    trainer.run_epochs(max(args.warmup, 1))
    barrier()

    # ---- timed region: K epochs, device events on the trainer's stream -------
    # Each epoch is one replay of the CUDA graph captured from an epoch
    # (kernels + NCCL collectives); the warm-up above ran the eager epoch and
    # the capture.
    launches0 = cg.kernel_launches()
    ledger0 = trainer.ledger()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        barrier()
        start.record(stream)
        for _ in range(args.steps):
            trainer.epoch_async()
        end.record(stream)
        barrier()
    launches = cg.kernel_launches() - launches0
    ledger1 = trainer.ledger()
    cost = None
    if world > 1:
        # The timed epochs' metered traffic of every rank against the analytic
        # model (compare_cost, cost.cpp:115-161) at the hidden width, which is
        # what the narrow-first panels carry.
        delta = torch.tensor([ledger1[c][f] - ledger0[c][f] for c in cg.CATEGORIES
                              for f in ("messages", "words_sent", "words_received", "payload_words",
                                        "calls")], dtype=torch.int64, device="cuda")
        allled = [torch.zeros_like(delta) for _ in range(world)]
        pg.all_gather(allled, delta)
        if rank == 0:
            leds = []
            for t in allled:
                v = t.cpu().numpy().tolist()
                leds.append({c: dict(zip(("messages", "words_sent", "words_received",
                                          "payload_words", "calls"), v[5 * i:5 * i + 5]))
                             for i, c in enumerate(cg.CATEGORIES)})
            try:
                cost = cg.compare_cost(strat, cg.CostParams(cfg["n"], data.nnz, cfg["dims"][1],
                                                            len(cfg["dims"]) - 1, N, repl),
                                       leds, args.steps)
                cost["f"] = cfg["dims"][1]
                cost["note"] = ("the model describes the reference schedule at one uniform width; "
                                "narrow-first panels, the real per-layer Y shapes and resident "
                                "SUMMA tiles move less, so only the reference schedule reconciles "
                                "exactly (tests/test_cost_model.py)")
            except Exception as e:  # pragma: no cover
                cost = {"unavailable": str(e)}
    # NVLink words received per rank per epoch (reference ledger conventions).
    recv_words = sum(ledger1[c]["words_received"] - ledger0[c]["words_received"]
                     for c in ledger1) / max(args.steps, 1)
    losses = trainer.losses()
    ms_total = start.elapsed_time(end)

    ms_t = torch.tensor([ms_total], dtype=torch.float64, device="cuda")
    if pg:
        pg.all_reduce(ms_t, op=pg.ReduceOp.MAX)
    ms_step = float(ms_t.item()) / args.steps

    # ---- profiled region: the same K epochs eager, CUDA events per kernel ----
    # (per-launch durations for the roofline; events cannot sit between the
    # kernels of a replayed graph without serialising it).
    trainer.set_timing(True)
    trainer.profile_reset()
    s1, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    s1.record(stream)
    for _ in range(args.steps):
        trainer.epoch_async()
    e1.record(stream)
    barrier()
    trainer.set_timing(False)
    prof = trainer.profile()
    ms_prof_total = s1.elapsed_time(e1)
    pt = torch.tensor([ms_prof_total], dtype=torch.float64, device="cuda")
    if pg:
        pg.all_reduce(pt, op=pg.ReduceOp.MAX)
    eager_ms_step = float(pt.item()) / args.steps
    trainer.run_epochs(2)  # re-capture the graph for what follows
    barrier()

    # ---- the other propagation order, same trainer, same timing rules --------
    alt = None
    if not args.no_alt:
        lib_set = cg.lib.cagnet_trainer_set_option
        cg.check(lib_set(trainer.h, b"reassociate", int(not strat.reassociate)))
        trainer.run_epochs(2)  # eager epoch + graph capture
        barrier()
        s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s2.record(stream)
        for _ in range(args.steps):
            trainer.epoch_async()
        e2.record(stream)
        barrier()
        alt_t = torch.tensor([s2.elapsed_time(e2)], dtype=torch.float64, device="cuda")
        if pg:
            pg.all_reduce(alt_t, op=pg.ReduceOp.MAX)
        alt = {"propagation": "reference order (A^T H) W" if strat.reassociate
               else "narrow-first A^T (H W)",
               "ms_per_step": round(float(alt_t.item()) / args.steps, 4)}
        cg.check(lib_set(trainer.h, b"reassociate", int(strat.reassociate)))

    # ---- end-to-end: the public host-buffer call, H2D + epoch + D2H ----------
    r0, r1, c0, c1, _ = trainer.tile(rank, cfg["dims"][0])
    feats = data.features()[r0:r1, c0:c1]
    x_pin = torch.empty(feats.shape, dtype=torch.float32, pin_memory=True)
    x_pin.numpy()[:] = feats
    lab_pin = torch.empty(r1 - r0, dtype=torch.int32, pin_memory=True)
    lab_pin.numpy()[:] = data.labels()[r0:r1]
    for _ in range(2):  # warm: eager epoch, then the graph capture
        trainer.step_host(x_pin.numpy(), lab_pin.numpy())
    barrier()
    # Synchronous steps: per-step wall time of step_host (copy -> epoch -> loss
    # D2H, nothing overlapped); the median keeps one host hiccup out.
    e2e_steps = []
    for _ in range(args.steps):
        t1 = time.perf_counter()
        trainer.step_host(x_pin.numpy(), lab_pin.numpy())
        e2e_steps.append((time.perf_counter() - t1) * 1e3)
    barrier()
    sync_ms = statistics.median(e2e_steps)
    sync_mean = statistics.mean(e2e_steps)
    # Pipelined steps (the headline e2e): prefetch_host queues step k+1's H2D
    # on a copy stream while step k's epoch runs; every step's copy and loss
    # D2H are inside the timed region, which spans all K steps.  One untimed
    # pipelined step first: the copy stream and the two staging slots are
    # created on first use (with peer access enabled, those allocations are
    # mapped into every peer and took 68 ms at 4 GPUs).
    trainer.prefetch_host(x_pin.numpy(), lab_pin.numpy())
    trainer.step_prefetched()
    trainer.prefetch_host(x_pin.numpy(), lab_pin.numpy())
    trainer.step_prefetched()
    barrier()
    t1 = time.perf_counter()
    trainer.prefetch_host(x_pin.numpy(), lab_pin.numpy())
    for k in range(args.steps):
        if k + 1 < args.steps:
            trainer.prefetch_host(x_pin.numpy(), lab_pin.numpy())
        trainer.step_prefetched()
    pipe_ms = (time.perf_counter() - t1) * 1e3 / args.steps
    barrier()
    e2e_t = torch.tensor([pipe_ms, sync_ms], dtype=torch.float64, device="cuda")
    if pg:
        pg.all_reduce(e2e_t, op=pg.ReduceOp.MAX)
    e2e_ms, sync_ms = float(e2e_t[0].item()), float(e2e_t[1].item())
    h2d = feats.size * 4 + (r1 - r0) * 4

    # ---- roofline of the dominant kernel (per-launch CUDA events) ------------
    dom_name, dom = max(prof.items(), key=lambda kv: kv[1]["ms"]) if prof else (None, None)
    peaks = load_peaks()
    peak = peaks.get("hbm_gbs", 6650.0)
    roof = None
    if dom:
        per_launch_ms = dom["ms"] / dom["launches"]
        bytes_per_launch = dom["bytes"] / dom["launches"]
        achieved = bytes_per_launch / (per_launch_ms * 1e-3) / 1e9
        roof = {"kernel": dom_name, "bound": "hbm", "achieved": round(achieved, 1),
                "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4),
                "traffic": load_traffic(dom_name),
                "bytes_per_launch": bytes_per_launch, "ms_per_launch": round(per_launch_ms, 4),
                # the kernel's device time per epoch over the graph-replayed epoch time
                "share_of_step": round(dom["ms"] / max(args.steps, 1) / max(ms_step, 1e-9), 4),
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback"}
        if dom_name.startswith("spmm_f"):
            # SURVEY 8(d)'s second byte model: every nonzero gathers one whole
            # f-wide row of H (no reuse), and the L1 wavefront floor of that
            # access pattern — one 128 B L1TEX wavefront per gathered row (the
            # rows are <= 64 B) plus one per 8 streamed {col, val} entries,
            # 148 SMs at the sampled SM clock.
            f = int(dom_name.split("_f")[1])
            rows = trainer.part_shape(0, 0)[0]  # every part of a rank spans its block rows
            nnz = sum(trainer.part_shape(0, q)[2] for q in range(trainer.num_parts()))
            gather = 8.0 * (rows + 1) + 8.0 * nnz + 4.0 * f * nnz + 4.0 * f * rows
            sm_hz = (clocks.summary().get("sm_mhz") or 1965) * 1e6
            lsu_floor_ms = nnz * (1.0 + 1.0 / 8.0) / (148 * sm_hz) * 1e3
            roof.update({"gather_bytes_per_launch": gather,
                         "gather_GBps": round(gather / (per_launch_ms * 1e-3) / 1e9, 1),
                         "lsu_floor_ms": round(lsu_floor_ms, 4),
                         "lsu_frac": round(lsu_floor_ms / per_launch_ms, 4),
                         "gather_model": "no-reuse bytes 8(r+1)+8nnz+4f*nnz+4fr; L1 floor = "
                                         "nnz*(1+1/8) wavefronts / (148 SMs x SM clock)"})

    # ---- epoch roofline (north star): the slower of this rank's kernel bytes at
    # HBM bandwidth and its received block bytes at NVLink bandwidth, max over ranks.
    hbm_bytes = sum(v["bytes"] for v in prof.values()) / max(args.steps, 1)
    link_bytes = recv_words * 4.0
    rb = torch.tensor([hbm_bytes, link_bytes], dtype=torch.float64, device="cuda")
    if pg:
        pg.all_reduce(rb, op=pg.ReduceOp.MAX)
    hbm_bytes, link_bytes = float(rb[0].item()), float(rb[1].item())
    link_peak, link_meas = 900.0, 470.0
    t_hbm = hbm_bytes / (peak * 1e9) * 1e3
    t_link = link_bytes / (link_peak * 1e9) * 1e3
    epoch_roof = {
        "hbm_bytes_per_rank": round(hbm_bytes), "link_bytes_per_rank": round(link_bytes),
        "t_hbm_ms": round(t_hbm, 4), "t_link_ms": round(t_link, 4),
        "bound": "hbm" if t_hbm >= t_link else "nvlink",
        "floor_ms": round(max(t_hbm, t_link), 4),
        "frac": round(max(t_hbm, t_link) / max(ms_step, 1e-9), 4),
        "link_peak_gbs": link_peak,
        "t_link_measured_ms": round(link_bytes / (link_meas * 1e9) * 1e3, 4),
        "link_measured_gbs": link_meas,
        "source": "hbm: algorithmic bytes of every profiled kernel per epoch (SURVEY 8d byte "
                  "model); link: ledger words_received x 4 B per epoch; NVLink 5 nominal "
                  "900 GB/s per direction, measured all-to-all push ingress ~470 GB/s "
                  "(profiles/r01_s4_micro_push_4gpu.txt)"}

    if rank != 0:
        if pg:
            pg.destroy_process_group()
        return

    cpu = None
    if N == 1 and not args.no_cpu_baseline and cfg["generator"] == "reference":
        try:
            threads = ref_threads()
            sess, setup = reference_session(cfg, threads)
            sec = sess.epoch()
            cpu = {"value": round(sec * 1e3, 1), "unit": "ms", "cores": threads,
                   "kind": "reference",
                   "sample": f"one epoch of the reference run_distributed 1D P={threads} rank "
                             f"threads on the full graph (n={cfg['n']}, nnz={setup['nnz']}); "
                             f"no extrapolation", "setup_s": setup}
            del sess
        except Exception as e:
            cpu = {"value": None, "unit": "ms", "cores": 1, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    clk = clocks.summary()
    line = {
        "metric": METRIC, "value": round(ms_step, 4), "unit": "ms", "n_gpus": N,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": cfg["label"], "strategy": kind, "ranks": N, "repl": repl,
                   "block": args.block,
                   "fuse": args.fuse, "cuda_graph": True,
                   "propagation": "narrow-first A^T (H W)" if strat.reassociate
                   else "reference order (A^T H) W",
                   "generator": cfg["generator"],
                   "l2": "inputs larger than L2 (CSR A+A^T and H0 > 126 MB)"},
        "e2e": {"value": round(e2e_ms, 4), "unit": "ms", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": 8,
                "stat": "K pipelined steps through the public host-buffer API (prefetch_host + "
                        "step_prefetched: each step's H2D from pinned memory overlaps the previous "
                        "step's epoch, each step's loss read back), wall time / K, max over ranks",
                "sync_ms": round(sync_ms, 4),
                "sync_stat": "median per-step wall time of step_host (copy, epoch, loss D2H in "
                             "sequence), max over ranks",
                "sync_mean_ms": round(sync_mean, 4)},
        "gpu_launches": int(launches),
        "eager_ms_per_step": round(eager_ms_step, 4),
        "roofline": roof,
        "epoch_roofline": epoch_roof,
        "cost_model": cost,
        "cpu_baseline": cpu,
        "clocks": clk,
        "kernels": {k: {"launches": v["launches"], "ms_per_launch": round(v["ms"] / v["launches"], 4),
                        "GBps": round(v["bytes"] / (v["ms"] * 1e-3) / 1e9, 1) if v["ms"] else None}
                    for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])},
        "other_propagation": alt,
        "loss_last": float(losses[-1]) if len(losses) else None,
        "setup_s": {"dataset_gen": round(gen_s, 2)},
    }
    if world > 1:
        line["parity"] = serial_parity(cg, data, cfg, strat, losses) if rank == 0 else None
    print(json.dumps(line))
    if pg:
        pg.destroy_process_group()


def serial_parity(cg, data, cfg, strat, losses, tol=1e-4):
    """Every multi-GPU bench run checks its own numbers: rank 0 trains a P = 1 trainer (the
    serial step, gnn.cpp:68-132) on its copy of the same graph, same initial weights, and
    compares the first epochs' losses with the distributed run's (the tolerance of the
    strategy-vs-serial tests, tests/test_gpu_training.py)."""
    k = int(min(len(losses), 4))
    if k == 0:
        return None
    serial = cg.make_trainer(data, cg.init_glorot(cfg["dims"], SEED_W, LR),
                             cg.Strategy("1d", 1, 1, reassociate=strat.reassociate, fuse=strat.fuse),
                             0, None)
    try:
        serial.distribute()
        serial.run_epochs(k)
        ref = np.asarray(serial.losses()[:k], dtype=np.float64)
    finally:
        serial.free()
    got = np.asarray(losses[:k], dtype=np.float64)
    rel = float(np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-30)))
    return {"vs": "P=1 trainer on rank 0, same graph and initial weights", "epochs": k,
            "max_rel": rel, "tol": tol, "ok": bool(rel <= tol)}


def main():
    args = parse()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
