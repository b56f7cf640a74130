"""Oracle parity at the headline size (BASELINE configs[1], Reddit-shaped:
232,965 vertices, ~115 M nonzeros), following verify_against_serial
(harness.cpp:118-166): the same dataset and model from the same seeds on both
sides, the same epochs, rel_frobenius (dense.cpp:190-201) <= 1e-4 on h_final
and every y_l, g_l, w_l, |dloss| / max(1, |loss|) <= 1e-4 per epoch, structure
bit-exact.

The reference side is the unmodified reference (oracle/_ref): make_dataset
(dataset.cpp:76-90) on the raw ER graph, then run_distributed 1D with one rank
per host thread (dist_common.cpp:205-222; the reference's thread-per-rank
model).  The raw graph comes from the oracle's multi-threaded restatement of
generate_erdos_renyi (csr.cpp:195-218, GF(2) jump-ahead of the row
sub-streams), and the first check is that the GPU's generator reproduces it
bit for bit — the whole 5.4e10-draw stream, not a sample.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N, E = 232965, 114848857
DIMS = [602, 16, 16, 41]
TOL = 1e-4


@pytest.fixture(scope="module")
def both(cg, orc, ref):
    threads = max(1, min(os.cpu_count() or 1, 64))
    raw = orc.er_generate_mt(N, E / N, 1, threads)
    x = orc.random_features(N, DIMS[0], 2)
    y = orc.random_labels(N, DIMS[-1], 3)
    rdata = ref.dataset_make(raw, x, y, DIMS[-1])
    del x, y
    gdata = cg.generate_dataset(N, E / N, DIMS[0], DIMS[-1], 1, 2, 3, device=0)
    yield raw, rdata, gdata, threads
    gdata.free()


def test_reddit_graph_bitexact(both):
    """GPU ER + normalize + transpose == the reference's, every array bit for bit."""
    raw, rdata, gdata, _ = both
    for which in (0, 1):
        rrp, rci, rv = gdata.csr(which).download()
        ref = rdata.csr(which)
        assert np.array_equal(rrp, ref.row_ptr)
        assert np.array_equal(rci.astype(np.int64), ref.col_idx)
        assert np.array_equal(rv, ref.vals.astype(np.float32))
    # The raw stream itself: adj minus its diagonal is the raw ER graph.
    rp, ci, _ = gdata.csr(0).download()
    deg = np.diff(rp)
    row = np.repeat(np.arange(N, dtype=np.int64), deg)
    off = ci.astype(np.int64) != row
    assert np.array_equal(ci[off].astype(np.int64), raw.col_idx)


@pytest.mark.parametrize("reassociate", [True, False])
def test_reddit_training_matches_reference(cg, ref, both, reassociate):
    """Two full-batch epochs on the GPU (1D, one rank; narrow-first and the
    reference's propagation order) against the reference's run_distributed."""
    raw, rdata, gdata, threads = both
    epochs = 2
    model = cg.init_glorot(DIMS, 4, 0.5)
    rmodel = ref.model(DIMS, 4, 0.5)
    for l in range(len(DIMS) - 1):
        assert np.array_equal(model.weights[l], rmodel.weights()[l])
    t = cg.make_trainer(gdata, model, cg.Strategy("1d", 1, reassociate=reassociate))
    t.distribute()
    losses = t.run_epochs(epochs)
    sess = ref.session(rdata, rmodel, "1d", threads)
    for _ in range(epochs):
        sess.epoch()
    out = sess.outcome()

    def rel(a, b):
        return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-300))

    errs = {"loss": max(abs(a - b) / max(1.0, abs(b)) for a, b in zip(losses, out.losses)),
            "h_final": rel(t.h_tile(len(DIMS) - 1), out.h_final)}
    for l in range(len(DIMS) - 1):
        errs[f"y{l}"] = rel(t.y(l), out.y[l])
        errs[f"w{l}"] = rel(t.weight(l), out.w[l])
        errs[f"g{l}"] = rel(t.g_tile(l), out.g[l])
    assert max(errs.values()) < TOL, errs
