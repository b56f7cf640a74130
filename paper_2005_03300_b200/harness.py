"""Experiment harness on B200s: the reference's ExperimentConfig / run_report /
verify_against_serial (harness.hpp:30-80, harness.cpp:22-166) over the GPU
trainers, emitting the same "cagnet-sim/1" report schema (config echo, loss
trace, result norms, per-category ledger) plus a "b200" section with device
timing.  The serial reference of verify_against_serial is this library's own
one-GPU 1D run (as in the reference, where it is its own serial path).

    python -m paper_2005_03300_b200.harness --n 4096 --degree 16 \\
        --dims 128,16,8 --strategy 2d --ranks 4 --epochs 5 [--verify 1e-4]
"""
from __future__ import annotations

import argparse
import json
import sys
from dataclasses import dataclass, field

import numpy as np

from . import api

SCHEMA = "cagnet-sim/1"


@dataclass
class ExperimentConfig:
    """harness.hpp:30-53 (scheduler dropped: NCCL replaces the simulator)."""
    n: int = 64
    degree: float = 8.0
    layer_dims: list = field(default_factory=lambda: [16, 16, 4])
    epochs: int = 5
    learning_rate: float = 0.5
    seed_graph: int = 1
    seed_features: int = 2
    seed_labels: int = 3
    seed_weights: int = 4
    seed_permutation: int = 5
    permute: bool = False
    serial: bool = False
    strategy: api.Strategy = field(default_factory=api.Strategy)
    edges_path: str = ""
    features_path: str = ""
    labels_path: str = ""
    undirected: bool = False
    generator: str = "reference"


def harness_dataset(cfg: ExperimentConfig, device: int = 0) -> api.GraphDataset:
    """harness.cpp:22-39 on `device`."""
    if len(cfg.layer_dims) < 2:
        raise api.InvalidArgument(1, "experiment: need at least two layer dims")
    paths = (cfg.edges_path, cfg.features_path, cfg.labels_path)
    if any(paths):
        if not all(paths):
            raise api.InvalidArgument(
                1, "experiment: edges, features and labels paths must be set together")
        data = api.load_dataset(*paths, undirected=cfg.undirected, device=device)
    else:
        data = api.generate_dataset(cfg.n, cfg.degree, cfg.layer_dims[0], cfg.layer_dims[-1],
                                    cfg.seed_graph, cfg.seed_features, cfg.seed_labels,
                                    device=device, generator=cfg.generator)
    if cfg.permute:
        data, _ = api.permute_random(data, cfg.seed_permutation)
    return data


def harness_model(cfg: ExperimentConfig, data: api.GraphDataset) -> api.GnnModel:
    """harness.cpp:41-45 (validate_model_against: widths match the dataset)."""
    if cfg.layer_dims[0] != data.num_features or cfg.layer_dims[-1] != data.num_classes:
        raise api.InvalidArgument(
            1, f"model: dims {cfg.layer_dims[0]}->{cfg.layer_dims[-1]} do not match the dataset "
               f"({data.num_features} features, {data.num_classes} classes)")
    return api.init_glorot(cfg.layer_dims, cfg.seed_weights, cfg.learning_rate)


def config_json(cfg: ExperimentConfig) -> dict:
    """harness.cpp:47-76."""
    j = {"n": cfg.n, "degree": cfg.degree, "layer_dims": list(cfg.layer_dims),
         "epochs": cfg.epochs, "learning_rate": cfg.learning_rate,
         "seeds": {"graph": cfg.seed_graph, "features": cfg.seed_features,
                   "labels": cfg.seed_labels, "weights": cfg.seed_weights,
                   "permutation": cfg.seed_permutation},
         "permute": cfg.permute, "scheduler": "nccl"}
    if cfg.serial:
        j["strategy"] = "serial"
    else:
        s = cfg.strategy
        j["strategy"] = {"kind": s.kind, "ranks": s.ranks, "repl": s.repl, "block": s.block}
    if cfg.edges_path:
        j["dataset_files"] = {"edges": cfg.edges_path, "features": cfg.features_path,
                              "labels": cfg.labels_path, "undirected": cfg.undirected}
    return j


def ledger_report(ledgers: list, strat: api.Strategy) -> dict:
    """ledger.cpp:100-125: per-category totals over ranks and the grid shape."""
    g = api.ProcessGrid(strat)
    per = {}
    for cat in api.CATEGORIES:
        tot = {k: 0 for k in ("messages", "words", "words_received", "payload_words", "calls")}
        for led in ledgers:
            c = led[cat]
            tot["messages"] += c["messages"]
            tot["words"] += c["words_sent"]
            tot["words_received"] += c["words_received"]
            tot["payload_words"] += c["payload_words"]
            tot["calls"] += c["calls"]
        per[cat] = tot
    return {"grid": {"kind": strat.kind, "ranks": g.ranks, "rows": g.rows, "cols": g.cols,
                     "layers": g.layers},
            "per_category": per}


def _frobenius(x) -> float:
    return float(np.sqrt(np.sum(np.square(np.asarray(x, np.float64)))))


def _serial_strategy(strat: api.Strategy) -> api.Strategy:
    return api.Strategy("1d", 1, 1, 0, reassociate=strat.reassociate, fuse=strat.fuse,
                        graph=strat.graph)


def _train_single(cfg: ExperimentConfig, strat: api.Strategy):
    data = harness_dataset(cfg, 0)
    model = harness_model(cfg, data)
    t = api.make_trainer(data, model, strat)
    t.distribute()
    losses = t.run_epochs(cfg.epochs)
    L = len(cfg.layer_dims)
    return dict(data=data, losses=np.asarray(losses),
                h_final=t.h_tile(L - 1).astype(np.float64),
                y=[t.y(l).astype(np.float64) for l in range(L - 1)],
                g=[t.g_tile(l).astype(np.float64) for l in range(L - 1)],
                w=[t.weight(l).astype(np.float64) for l in range(L - 1)],
                epoch_ms=t.last_epoch_ms())


def run_report(cfg: ExperimentConfig) -> dict:
    """harness.cpp:88-116: trains per the config and returns the report."""
    report = {"schema": SCHEMA, "config": config_json(cfg)}
    if cfg.serial:
        r = _train_single(cfg, _serial_strategy(cfg.strategy))
        data = r["data"]
        report["dataset"] = {"n": data.n, "nnz": data.nnz, "train_count": data.train_count(),
                             "num_classes": data.num_classes}
        report["losses"] = [float(x) for x in r["losses"]]
        report["final_loss"] = float(r["losses"][-1])
        report["h_final_norm"] = _frobenius(r["h_final"])
        report["weight_norms"] = [_frobenius(w) for w in r["w"]]
        report["b200"] = {"last_epoch_ms": r["epoch_ms"], "ranks": 1}
        return report
    out = api.run_distributed(lambda dev: harness_dataset(cfg, dev),
                              harness_model(cfg, harness_dataset(cfg, 0)), cfg.strategy,
                              cfg.epochs)
    data = harness_dataset(cfg, 0)
    report["dataset"] = {"n": data.n, "nnz": data.nnz, "train_count": data.train_count(),
                         "num_classes": data.num_classes}
    report["losses"] = [float(x) for x in out.losses]
    report["final_loss"] = float(out.losses[-1])
    report["h_final_norm"] = _frobenius(out.h_final)
    report["weight_norms"] = [_frobenius(w) for w in out.model.weights]
    report["ledger"] = ledger_report(out.ledger, cfg.strategy)
    report["prereduction_totals"] = [int(x) for x in out.prereduction_totals]
    report["memory_peaks"] = [int(x) for x in out.memory_peaks]
    s = cfg.strategy
    # B200 extension: the metered traffic against the analytic model
    # (compare_cost, cost.cpp:115-161) at the config's widest layer.
    params = api.CostParams(data.n, data.nnz, max(cfg.layer_dims), len(cfg.layer_dims) - 1, s.ranks,
                            s.repl)
    try:
        report["cost_model"] = api.compare_cost(s, params, out.ledger, cfg.epochs)
    except api.CagnetError as e:
        report["cost_model"] = {"unavailable": str(e)}
    report["b200"] = {"last_epoch_ms": out.epoch_ms, "ranks": s.ranks,
                      "reassociate": s.reassociate, "fuse": s.fuse, "cuda_graph": s.graph,
                      "p2p": s.p2p, "resident_sparse": s.resident_sparse}
    return report


def _rel(a, b) -> float:
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    nb = np.sqrt(np.sum(b * b))
    d = np.sqrt(np.sum((a - b) ** 2))
    return float(d / nb) if nb > 0 else float(d)


def verify_against_serial(cfg: ExperimentConfig, tolerance: float) -> dict:
    """harness.cpp:118-166: the partitioned run against the one-GPU run of the
    same dataset and model (relative Frobenius on h_final, y, g, w; absolute
    loss trace difference)."""
    if cfg.serial:
        raise api.InvalidArgument(1, "verify: pick a partitioned strategy to compare")
    ser = _train_single(cfg, _serial_strategy(cfg.strategy))
    model0 = harness_model(cfg, ser["data"])
    out = api.run_distributed(lambda dev: harness_dataset(cfg, dev), model0, cfg.strategy,
                              cfg.epochs)
    errors = {"h_final": _rel(out.h_final, ser["h_final"])}
    for l in range(len(cfg.layer_dims) - 1):
        errors[f"y_{l}"] = _rel(out.y_final[l], ser["y"][l])
        errors[f"g_{l}"] = _rel(out.g_final[l], ser["g"][l])
        errors[f"w_{l}"] = _rel(out.model.weights[l], ser["w"][l])
    errors["loss_trace"] = float(np.max(np.abs(np.asarray(out.losses) - ser["losses"])))
    worst = max(errors.values())
    return {"schema": SCHEMA, "config": config_json(cfg), "tolerance": tolerance,
            "max_rel_error": worst, "errors": errors, "pass": worst < tolerance}


def main(argv=None) -> int:
    p = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    p.add_argument("--n", type=int, default=64)
    p.add_argument("--degree", type=float, default=8.0)
    p.add_argument("--dims", default="16,16,4")
    p.add_argument("--epochs", type=int, default=5)
    p.add_argument("--lr", type=float, default=0.5)
    p.add_argument("--seeds", default="1,2,3,4,5", help="graph,features,labels,weights,perm")
    p.add_argument("--permute", action="store_true")
    p.add_argument("--serial", action="store_true")
    p.add_argument("--strategy", default="1d", choices=["1d", "1.5d", "2d", "3d"])
    p.add_argument("--ranks", type=int, default=1)
    p.add_argument("--repl", type=int, default=1)
    p.add_argument("--block", type=int, default=0)
    p.add_argument("--reference-order", action="store_true")
    p.add_argument("--edges")
    p.add_argument("--features")
    p.add_argument("--labels")
    p.add_argument("--undirected", action="store_true")
    p.add_argument("--verify", type=float, default=None, help="tolerance: run verify instead")
    a = p.parse_args(argv)
    sg, sf, sl, sw, sp = (int(x) for x in a.seeds.split(","))
    cfg = ExperimentConfig(
        n=a.n, degree=a.degree, layer_dims=[int(x) for x in a.dims.split(",")], epochs=a.epochs,
        learning_rate=a.lr, seed_graph=sg, seed_features=sf, seed_labels=sl, seed_weights=sw,
        seed_permutation=sp, permute=a.permute, serial=a.serial,
        strategy=api.Strategy(a.strategy, a.ranks, a.repl, a.block,
                              reassociate=not a.reference_order),
        edges_path=a.edges or "", features_path=a.features or "", labels_path=a.labels or "",
        undirected=a.undirected)
    if a.verify is not None:
        res = verify_against_serial(cfg, a.verify)
        print(json.dumps(res, indent=1))
        return 0 if res["pass"] else 1
    print(json.dumps(run_report(cfg), indent=1))
    return 0


if __name__ == "__main__":
    sys.exit(main())
