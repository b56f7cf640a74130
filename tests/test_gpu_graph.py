"""GPU CSR / block construction (K4) — bit-exact structure against the oracle
and the reference fixtures; values equal (float) of the reference fp64."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(autouse=True)
def _gpu(need_gpus):
    need_gpus(1)


@pytest.mark.parametrize("n,d,seed", [(32, 8.0, 1), (64, 8.0, 7), (20, 4.0, 5), (1, 0.0, 3),
                                      (257, 30.0, 11), (4096, 16.0, 1)])
def test_er_generator_bitwise(cg, orc, n, d, seed):
    a = cg.generate_erdos_renyi(n, d, seed)
    rp, ci, v = a.download()
    o = orc.er_generate(n, d, seed)
    assert np.array_equal(rp, o.row_ptr)
    assert np.array_equal(ci, o.col_idx)
    assert np.all(v == 1.0)


def test_er_pinned_counts_on_gpu(cg):
    assert cg.generate_erdos_renyi(32, 8.0, 1).nnz == 249
    assert cg.generate_erdos_renyi(64, 8.0, 7).nnz == 495


def test_er_dense_probability_one(cg, orc):
    a = cg.generate_erdos_renyi(9, 9.0, 2)  # p = 1: complete graph without loops
    assert a.nnz == 72
    assert np.array_equal(a.download()[1], orc.er_generate(9, 9.0, 2).col_idx)


def test_normalize_transpose_bitwise(cg, orc):
    raw = cg.generate_erdos_renyi(300, 12.0, 4)
    adj = cg.add_self_loops_and_normalize(raw)
    o = orc.normalize(orc.er_generate(300, 12.0, 4))
    rp, ci, v = adj.download()
    assert np.array_equal(rp, o.row_ptr) and np.array_equal(ci, o.col_idx)
    assert np.array_equal(v, o.vals.astype(np.float32))
    t = cg.transpose(adj)
    ot = orc.transpose(o)
    rp, ci, v = t.download()
    assert np.array_equal(rp, ot.row_ptr) and np.array_equal(ci, ot.col_idx)
    assert np.array_equal(v, ot.vals.astype(np.float32))


def test_normalize_existing_diagonal(cg, orc):
    # test_sparse_core.cpp:91-95 — an existing diagonal is not duplicated.
    a = cg.csr_upload([0, 2, 3, 3], [0, 1, 2], 3)
    s = cg.add_self_loops_and_normalize(a)
    o = orc.normalize(orc.from_edge_list(3, [0, 0, 1], [0, 1, 2]))
    rp, ci, v = s.download()
    assert s.nnz == 5 and np.array_equal(ci, o.col_idx)
    assert np.array_equal(v, o.vals.astype(np.float32))


def test_extract_block_bitwise(cg, orc):
    o = orc.normalize(orc.er_generate(101, 9.0, 8))
    adj = cg.add_self_loops_and_normalize(cg.generate_erdos_renyi(101, 9.0, 8))
    for (r0, r1, c0, c1) in [(0, 101, 0, 101), (10, 40, 5, 77), (0, 0, 0, 101), (50, 51, 0, 0),
                             (34, 68, 68, 101), (100, 101, 99, 101)]:
        b = cg.extract_block(adj, r0, r1, c0, c1)
        ob = orc.extract_block(o, r0, r1, c0, c1)
        rp, ci, v = b.download()
        assert np.array_equal(rp, ob.row_ptr) and np.array_equal(ci, ob.col_idx)
        assert np.array_equal(v, ob.vals.astype(np.float32))
    with pytest.raises(cg.InvalidArgument):
        cg.extract_block(adj, 5, 3, 0, 101)


def test_dataset_generate_bitwise_config1(cg):
    c = np.load(os.path.join(GOLD, "reference_config1.npz"))
    d = cg.generate_dataset(4096, 16.0, 128, 8, 1, 2, 3)
    assert d.nnz == 70023 and d.train_count() == 4096
    rp, ci, v = d.adj.download()
    assert np.array_equal(rp, c["adj_row_ptr"]) and np.array_equal(ci, c["adj_col_idx"])
    assert np.array_equal(v, c["adj_vals"].astype(np.float32))
    rpt, cit, _ = d.adj_t.download()
    assert np.array_equal(rpt, c["adjt_row_ptr"]) and np.array_equal(cit, c["adjt_col_idx"])
    assert np.array_equal(d.features()[:64], c["features_head"].astype(np.float32))
    assert np.array_equal(d.labels(), c["labels"])


def test_dataset_features_bitwise(cg, orc):
    # U[0,1) draws through the GF(2) jump-ahead: (float) of the reference doubles.
    d = cg.generate_dataset(700, 5.0, 37, 3, 9, 10, 11)
    x = orc.random_features(700, 37, 10).astype(np.float32)
    assert np.array_equal(d.features(), x)
    assert np.array_equal(d.labels(), orc.random_labels(700, 3, 11))


def test_partition_blocks_match_reference(cg, orc):
    """Survey §7 minimum slice: per-rank block structure of the reference's
    distribute() (1D P=8, 2D P=4, 3D P=8, 1.5D P=8 c=2) on config 1,
    extracted on the GPU with the geometry of the product's grids."""
    c = np.load(os.path.join(GOLD, "reference_config1.npz"))
    d = cg.generate_dataset(4096, 16.0, 128, 8, 1, 2, 3)
    adj, adjt = d.adj, d.adj_t
    n = 4096
    for kind, P, repl in (("1d", 8, 1), ("2d", 4, 1), ("3d", 8, 1), ("1.5d", 8, 2)):
        grid = cg.ProcessGrid(cg.Strategy(kind, P, repl))
        want = c[f"parts_{kind}_p{P}"]
        got = []
        for r in range(P):
            if kind in ("1d", "1.5d"):
                r0, r1 = grid.tile(n, r, 1)[:2]
                blocks = grid.rows
                cols = [cg.block_range(n, blocks, q) for q in range(blocks)]
            else:
                i = (r % (grid.rows * grid.cols)) // grid.cols
                j = r % grid.cols
                k = r // (grid.rows * grid.cols)
                r0, r1 = cg.block_range(n, grid.rows, i)
                ob, oe = cg.block_range(n, grid.rows, j)
                ib, ie = cg.block_range(oe - ob, grid.layers, k)
                cols = [(ob + ib, ob + ie)]
            for q, (c0, c1) in enumerate(cols):
                got.append([r, q, cg.extract_block(adj, r0, r1, c0, c1).nnz,
                            cg.extract_block(adjt, r0, r1, c0, c1).nnz])
        assert np.array_equal(np.asarray(got), want), kind
    at1d = c["parts_1d_p8"][:, 3].reshape(8, 8).sum(axis=1)
    assert list(at1d) == [8794, 8929, 8874, 8640, 8852, 8733, 8640, 8561]
    at2d = c["parts_2d_p4"][:, 3]
    assert list(at2d) == [18595, 16642, 16405, 18381]
    at3d = c["parts_3d_p8"][:, 3]
    assert list(at3d) == [9330, 8297, 8246, 9141, 9265, 8345, 8159, 9240]


def test_skip_generator_properties(cg):
    n, deg = 20000, 16.0
    d = cg.generate_dataset(n, deg, 4, 3, 1, 2, 3, generator="skip")
    rp, ci, v = d.adj.download()
    raw_nnz = d.nnz - n
    assert abs(raw_nnz / n - deg) < 0.5
    for i in range(0, n, 997):
        cols = ci[rp[i]:rp[i + 1]]
        assert np.all(np.diff(cols) > 0) and i in cols
    d2 = cg.generate_dataset(n, deg, 4, 3, 1, 2, 3, generator="skip")
    assert np.array_equal(d2.adj.download()[1], ci)
