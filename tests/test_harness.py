"""Experiment harness (harness.hpp:30-80): run_report / verify_against_serial
over the GPU trainers, reference "cagnet-sim/1" schema."""
import json

import numpy as np
import pytest

PINNED = [1.4676915537761182, 1.3547714828994135, 1.3527671034478277,
          1.3514914086563463, 1.3507757616337233]  # test_gnn_reference.cpp:148-164


def test_config_and_ledger_json_cpu(cg):
    from paper_2005_03300_b200 import harness
    cfg = harness.ExperimentConfig(strategy=cg.Strategy("2d", 4, 1, 3))
    j = harness.config_json(cfg)
    assert j["strategy"] == {"kind": "2d", "ranks": 4, "repl": 1, "block": 3}
    assert j["seeds"] == {"graph": 1, "features": 2, "labels": 3, "weights": 4, "permutation": 5}
    zero = {c: {k: 1 for k in ("messages", "words_sent", "words_received", "payload_words",
                               "calls")} for c in cg.CATEGORIES}
    rep = harness.ledger_report([zero] * 4, cfg.strategy)
    assert rep["grid"] == {"kind": "2d", "ranks": 4, "rows": 2, "cols": 2, "layers": 1}
    assert rep["per_category"]["dbcast"] == {"messages": 4, "words": 4, "words_received": 4,
                                             "payload_words": 4, "calls": 4}
    json.dumps(rep)


@pytest.mark.gpu
def test_run_report_serial_pinned_trace(cg, need_gpus):
    need_gpus(1)
    from paper_2005_03300_b200 import harness
    cfg = harness.ExperimentConfig(n=32, degree=8.0, layer_dims=[16, 16, 4], epochs=5,
                                   learning_rate=0.5, serial=True)
    rep = harness.run_report(cfg)
    assert rep["schema"] == "cagnet-sim/1" and rep["dataset"]["nnz"] == 281
    for a, b in zip(rep["losses"], PINNED):
        assert abs(a - b) / max(1.0, abs(b)) < 1e-4
    assert rep["b200"]["last_epoch_ms"] > 0
    json.dumps(rep)


@pytest.mark.gpu
@pytest.mark.parametrize("kind,P", [("1d", 1), ("2d", 1), ("3d", 1), ("1d", 2), ("2d", 4)])
def test_verify_against_serial(cg, need_gpus, kind, P):
    need_gpus(P)
    from paper_2005_03300_b200 import harness
    cfg = harness.ExperimentConfig(n=90, degree=6.0, layer_dims=[24, 8, 6], epochs=3,
                                   strategy=cg.Strategy(kind, P, 1, 0, reassociate=True),
                                   permute=True)
    res = harness.verify_against_serial(cfg, 1e-4)
    assert res["pass"], res["errors"]
    rep = harness.run_report(cfg)
    assert rep["ledger"]["grid"]["ranks"] == P
    if P > 1:
        assert rep["ledger"]["per_category"]["dbcast"]["calls"] > 0


@pytest.mark.gpu
def test_harness_cli(cg, need_gpus, capsys):
    need_gpus(1)
    from paper_2005_03300_b200 import harness
    assert harness.main(["--n", "40", "--dims", "8,6,3", "--epochs", "2", "--verify", "1e-4",
                         "--strategy", "2d"]) == 0
    out = json.loads(capsys.readouterr().out)
    assert out["pass"] is True
