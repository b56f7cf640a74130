"""Analytic communication model (cost.hpp / cost.cpp of the reference):
pinned spot values from the reference's own tests (test_cost_model.cpp,
acceptance_test.cpp:349-371) on CPU, and the reconciliation of real B200
runs' metered ledgers with it (test_dist_strategies.cpp:280-347) on a GPU."""
import numpy as np
import pytest

BASE = dict(n=1000, nnz=8000, f=32, layers=3, ranks=4, repl=1)


def test_ceil_lg(cg):
    assert [cg.ceil_lg(p) for p in (1, 2, 3, 4, 5, 8, 9, 1024, 1025)] == [0, 1, 2, 2, 3, 3, 4, 10, 11]
    with pytest.raises(cg.InvalidArgument):
        cg.ceil_lg(0)


def test_cost_spot_values(cg):
    p = cg.predict_cost("1d", cg.CostParams(**BASE))
    assert (p["words"], p["messages"]) == (195072, 30)
    assert p["terms"] == {"embedding_broadcast": 192000, "weight_gradient_reduce": 3072}
    q = cg.predict_cost("1.5d", cg.CostParams(**{**BASE, "repl": 2}))
    assert (q["words"], q["messages"]) == (192000, 18)
    assert cg.predict_cost("1.5d", cg.CostParams(**BASE))["words"] == 3 * (2 * 1000 * 32 + 2 * 1000 * 32 // 4)
    t = cg.predict_cost("2d", cg.CostParams(**{**BASE, "ranks": 16}))
    assert (t["words"], t["messages"]) == (207072, 72)
    c = cg.predict_cost("3d", cg.CostParams(**{**BASE, "ranks": 8}))
    assert (c["words"], c["messages"]) == (300000, 24)
    for pred in (p, q, t, c):
        assert sum(pred["terms"].values()) == pred["words"]


def test_cost_rejects_impossible_shapes(cg):
    for kind, over in (("1d", {"n": 0}), ("1d", {"ranks": 0}), ("2d", {"ranks": 5}),
                       ("3d", {"ranks": 6}), ("1.5d", {"repl": 3}), ("1d", {"layers": 0})):
        with pytest.raises(cg.InvalidArgument):
            cg.predict_cost(kind, cg.CostParams(**{**BASE, **over}))


def test_rect_layer_and_footprints(cg):
    p = cg.CostParams(n=100, nnz=500, f=8, layers=3, ranks=4)
    assert cg.predict_2d_rect_layer(p, 4, 6, 1.0, 0.0) == 2.0
    beta = cg.predict_2d_rect_layer(p, 4, 6, 0.0, 1.0)
    assert beta == pytest.approx(500 / 4 + 800 / 6 + 800 / 4, rel=1e-15)
    assert cg.predict_2d_rect_layer(p, 4, 6, 2.0, 0.5) == pytest.approx(2 * 2.0 + 0.5 * beta, rel=1e-15)
    with pytest.raises(cg.InvalidArgument):
        cg.predict_2d_rect_layer(p, 0, 6, 1.0, 1.0)
    m = cg.memory_footprints(100, 500, 8, 8, 3, 2, 8)
    assert m == {"serial": 2900, "repl15d": 7800, "repl15d_single_adj": 5800, "split3d_peak": 3700}
    with pytest.raises(cg.InvalidArgument):
        cg.memory_footprints(100, 500, 8, 8, 1, 2, 8)
    with pytest.raises(cg.InvalidArgument):
        cg.memory_footprints(100, 500, 8, 8, 3, 2, 6)


def _ledgers(P, dbcast):
    z = {f: 0 for f in ("messages", "words_sent", "words_received", "payload_words", "calls")}
    out = []
    for r in range(P):
        led = {c: dict(z) for c in ("dbcast", "sbcast", "reduce", "allgather")}
        led["dbcast"]["payload_words"] = dbcast[r]
        out.append(led)
    return out


def test_compare_cost_synthetic(cg):
    strat = cg.Strategy("1d", 4)
    words = cg.predict_cost("1d", cg.CostParams(**BASE))["words"]
    cmp = cg.compare_cost(strat, cg.CostParams(**BASE), _ledgers(4, [words + 1] * 4), 1)
    assert cmp["exact"] and cmp["within_band"] and cmp["ratio"] == 1.0
    assert (cmp["predicted_words"], cmp["extra_words"], cmp["strategy"]) == (words, 1, "1d")
    off = cg.compare_cost(strat, cg.CostParams(**BASE), _ledgers(4, [words + 5] + [words + 1] * 3), 1)
    assert not off["within_band"]
    one = cg.compare_cost(cg.Strategy("1d", 1), cg.CostParams(**{**BASE, "ranks": 1}), _ledgers(1, [0]), 3)
    assert one["degenerate"] and one["within_band"] and one["measured_words"] == 0.0


@pytest.mark.gpu
@pytest.mark.parametrize("kind,P,repl,n", [("1d", 4, 1, 64), ("1.5d", 8, 2, 96), ("2d", 4, 1, 32),
                                           ("3d", 8, 1, 32)])
def test_b200_traffic_reconciles_with_model(cg, need_gpus, kind, P, repl, n):
    """The metered traffic of real runs (reference schedule) against the
    closed forms: exact for 1D / 1.5D, inside [0.5, 2] for 2D / 3D."""
    need_gpus(1)
    data = cg.generate_dataset(n, 6.0, 16, 16, 1, 2, 3, device=0)
    model = cg.init_glorot([16, 16, 16], 4, 0.5)
    strat = cg.Strategy(kind, P, repl, resident_sparse=False)
    out = cg.run_distributed(data, model, strat, 2)
    cmp = cg.compare_cost(strat, cg.CostParams(n, data.nnz, 16, 2, P, repl), out.ledger, 2)
    assert cmp["within_band"] and not cmp["degenerate"], cmp
    if kind in ("1d", "1.5d"):
        assert cmp["exact"] and cmp["ratio"] == 1.0, cmp
    else:
        assert 0.5 <= cmp["ratio"] <= 2.0, cmp
