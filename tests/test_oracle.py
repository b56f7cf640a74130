"""The CPU oracle (oracle/cagnet_oracle.c) pinned against the reference's own
golden vectors (proj/tests/*.cpp) and against the reference itself
(oracle/_ref, or the committed fixtures generated from it)."""
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return np.load(os.path.join(GOLD, name))


# test_sparse_core.cpp:155-172
def test_er_pinned_counts(orc):
    assert orc.er_generate(32, 8.0, 1).nnz == 249
    assert orc.er_generate(64, 8.0, 7).nnz == 495
    g = orc.er_generate(32, 8.0, 1)
    for i in range(32):
        cols = g.col_idx[g.row_ptr[i]:g.row_ptr[i + 1]]
        assert i not in cols
        assert np.all(np.diff(cols) > 0)
    assert not np.array_equal(orc.er_generate(32, 8.0, 2).col_idx[:50], g.col_idx[:50])


def test_er_matches_reference_fixture(orc):
    gd = load("reference_small.npz")
    for key in ("er_32_8_1", "er_64_8_7", "er_20_4_5"):
        _, n, d, s = key.split("_")
        a = orc.er_generate(int(n), float(d), int(s))
        assert np.array_equal(a.row_ptr, gd[key + "_row_ptr"])
        assert np.array_equal(a.col_idx, gd[key + "_col_idx"])


def test_er_multithreaded_equals_sequential(orc):
    """The jump-ahead restatement (row sub-streams at draw u*(n-1)) reproduces
    the sequential generator bit for bit, for any thread count."""
    for n, d, s, t in ((32, 8.0, 1, 3), (64, 8.0, 7, 8), (2500, 9.0, 11, 5)):
        a, b = orc.er_generate(n, d, s), orc.er_generate_mt(n, d, s, t)
        assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col_idx, b.col_idx)
    assert orc.er_generate_mt(32, 8.0, 1, 4).nnz == 249  # test_sparse_core.cpp:163


def test_rng_jump_ahead(orc):
    seq = orc.rng_draws(9, 0, 600)
    for k in (1, 63, 64, 65, 599):
        assert np.array_equal(orc.rng_draws(9, k, 600 - k), seq[k:])


def test_er_multithreaded_matches_live_reference(orc, ref):
    a, b = ref.er(1500, 12.0, 3), orc.er_generate_mt(1500, 12.0, 3, 6)
    assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col_idx, b.col_idx)


# test_sparse_core.cpp:39-55
def test_from_edge_list_golden(orc):
    a = orc.from_edge_list(3, [0, 0, 2], [1, 1, 0], undirected=False)
    assert list(a.row_ptr) == [0, 1, 1, 2] and list(a.col_idx) == [1, 0]
    u = orc.from_edge_list(3, [0, 0, 2], [1, 1, 0], undirected=True)
    assert list(u.row_ptr) == [0, 2, 3, 4] and list(u.col_idx) == [1, 2, 0, 0]
    with pytest.raises(ValueError):
        orc.from_edge_list(3, [0], [3])


# test_sparse_core.cpp:74-96
def test_normalize_hand_oracle(orc):
    a = orc.from_edge_list(3, [0, 1], [1, 2])
    s = orc.normalize(a)
    assert s.nnz == 5
    d = np.zeros((3, 3))
    for i in range(3):
        for k in range(s.row_ptr[i], s.row_ptr[i + 1]):
            d[i, s.col_idx[k]] = s.vals[k]
    assert d[0, 0] == pytest.approx(0.5, rel=1e-15)
    assert d[0, 1] == pytest.approx(0.5, rel=1e-15)
    assert d[1, 1] == pytest.approx(0.5, rel=1e-15)
    assert d[1, 2] == pytest.approx(1 / np.sqrt(2), rel=1e-15)
    assert d[2, 2] == pytest.approx(1.0, rel=1e-15)
    assert d[1, 0] == d[2, 0] == d[2, 1] == 0.0
    s2 = orc.normalize(orc.from_edge_list(3, [0, 0, 1], [0, 1, 2]))
    assert s2.nnz == 5 and np.array_equal(s2.col_idx, s.col_idx) and np.array_equal(s2.vals, s.vals)


# test_sparse_core.cpp:98-108, 110-128
def test_transpose_and_extract_golden(orc):
    a = orc.from_edge_list(3, [0, 0, 2], [1, 2, 1])
    t = orc.transpose(a)
    assert list(t.row_ptr) == [0, 0, 2, 3] and list(t.col_idx) == [0, 2, 0]
    tt = orc.transpose(t)
    assert np.array_equal(tt.row_ptr, a.row_ptr) and np.array_equal(tt.col_idx, a.col_idx)
    b = orc.from_edge_list(4, [0, 1, 2, 3], [1, 3, 0, 2])
    blk = orc.extract_block(b, 1, 3, 2, 4)
    assert list(blk.row_ptr) == [0, 1, 1] and list(blk.col_idx) == [1]
    big = orc.er_generate(17, 5.0, 3)
    total = sum(orc.extract_block(big, 0, 17, *orc.block_range(17, 4, q)).nnz for q in range(4))
    assert total == big.nnz


# test_dist.cpp:102-104
def test_block_sizes_golden(orc):
    def sizes(n, p):
        return [e - b for b, e in (orc.block_range(n, p, i) for i in range(p))]
    assert sizes(10, 4) == [3, 3, 3, 1]
    assert sizes(3, 4) == [1, 1, 1, 0]
    assert sizes(12, 3) == [4, 4, 4]


# test_sparse_core.cpp:130-153: SpMM equals the dense product, column splits compose bitwise.
def test_spmm_column_split_bitwise(orc):
    a = orc.normalize(orc.er_generate(19, 6.0, 9))
    h = orc.random_features(19, 7, 10)
    whole = orc.spmm(a, h)
    dense = np.zeros((19, 19))
    for i in range(19):
        for k in range(a.row_ptr[i], a.row_ptr[i + 1]):
            dense[i, a.col_idx[k]] = a.vals[k]
    assert np.allclose(whole, dense @ h, rtol=0, atol=1e-14)
    for parts in (2, 3, 5):
        acc = np.zeros((19, 7))
        for q in range(parts):
            c0, c1 = orc.block_range(19, parts, q)
            piece = orc.extract_block(a, 0, 19, c0, c1)
            acc = orc.spmm(piece, h[c0:c1], acc)
        assert np.array_equal(acc, whole)


# test_gnn_reference.cpp:148-164 — the pinned loss trace, exact.
def test_pinned_loss_trace(orc):
    expected = [1.4676915537761182, 1.3547714828994135, 1.3527671034478277,
                1.3514914086563463, 1.3507757616337233]
    data = orc.generate_dataset(32, 8.0, 16, 4, 1, 2, 3)
    assert data["adj"].nnz == 281
    w = orc.init_glorot([16, 16, 4], 4)
    losses, h, y, g, wf = orc.train_serial(data, [16, 16, 4], w, 0.5, 5)
    assert list(losses) == expected


def test_oracle_bitwise_equals_reference_fixture(orc):
    gd = load("reference_small.npz")
    data = orc.generate_dataset(32, 8.0, 16, 4, 1, 2, 3)
    assert np.array_equal(data["adj"].row_ptr, gd["ds32_adj_row_ptr"])
    assert np.array_equal(data["adj"].vals, gd["ds32_adj_vals"])
    assert np.array_equal(data["adj_t"].col_idx, gd["ds32_adjt_col_idx"])
    assert np.array_equal(data["adj_t"].vals, gd["ds32_adjt_vals"])
    assert np.array_equal(data["features"], gd["ds32_features"])
    assert np.array_equal(data["labels"], gd["ds32_labels"])
    w = orc.init_glorot([16, 16, 4], 4)
    for l in range(2):
        assert np.array_equal(w[l], gd[f"ds32_w0_{l}"])
    losses, h, y, g, wf = orc.train_serial(data, [16, 16, 4], w, 0.5, 5)
    assert np.array_equal(losses, gd["ds32_losses"])
    assert np.array_equal(h, gd["ds32_h_final"])
    for l in range(2):
        assert np.array_equal(y[l], gd[f"ds32_y_{l}"])
        assert np.array_equal(g[l], gd[f"ds32_g_{l}"])
        assert np.array_equal(wf[l], gd[f"ds32_w_{l}"])


def test_oracle_config1_structure(orc):
    c = load("reference_config1.npz")
    data = orc.generate_dataset(4096, 16.0, 128, 8, 1, 2, 3)
    assert data["adj"].nnz == 70023
    assert np.array_equal(data["adj"].row_ptr, c["adj_row_ptr"])
    assert np.array_equal(data["adj"].col_idx, c["adj_col_idx"])
    assert np.array_equal(data["adj"].vals, c["adj_vals"])
    assert np.array_equal(data["adj_t"].col_idx, c["adjt_col_idx"])
    assert np.array_equal(data["labels"], c["labels"])
    # Survey §7 minimum-slice pins: per-block nnz of the reference partitions.
    at = data["adj_t"]
    nnz_1d = [orc.extract_block(at, *orc.block_range(4096, 8, r), *orc.block_range(4096, 8, q)).nnz
              for r in range(8) for q in range(8)]
    per_rank = np.asarray(nnz_1d).reshape(8, 8).sum(axis=1)
    assert list(per_rank) == [8794, 8929, 8874, 8640, 8852, 8733, 8640, 8561]
    parts = c["parts_1d_p8"]
    assert list(parts[:, 3]) == nnz_1d


def test_oracle_matches_live_reference(orc, ref):
    data = ref.dataset(64, 8.0, 12, 5, 7, 8, 9)
    od = orc.generate_dataset(64, 8.0, 12, 5, 7, 8, 9)
    a = data.csr(0)
    assert np.array_equal(a.row_ptr, od["adj"].row_ptr)
    assert np.array_equal(a.vals, od["adj"].vals)
    model = ref.model([12, 10, 7, 5], 3, 0.25)
    res = ref.serial(data, model, 3)
    losses, h, y, g, w = orc.train_serial(od, [12, 10, 7, 5], model.weights(), 0.25, 3)
    assert np.array_equal(losses, res.losses)
    assert np.array_equal(h, res.h_final)
    for l in range(3):
        assert np.array_equal(y[l], res.y[l]) and np.array_equal(g[l], res.g[l])
