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


def test_er_generator_bitwise_past_2_32_draws(cg, orc):
    """n = 65,536: rows start at draw offsets up to 4.29e9 (> 2^32), so every
    high power of the GPU's GF(2) jump-ahead is exercised; compared with the
    oracle's SEQUENTIAL generator (one stream, no jumps)."""
    n, d, seed = 65536, 10.0, 17
    rp, ci, _ = cg.generate_erdos_renyi(n, d, seed).download()
    o = orc.er_generate(n, d, seed)
    assert np.array_equal(rp, o.row_ptr)
    assert np.array_equal(ci, o.col_idx)


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


@pytest.mark.parametrize("n,d,seed", [(200, 6.0, 77), (1000, 20.0, 5), (1, 0.0, 3)])
def test_permute_random_bitwise(cg, ref, n, d, seed):
    """permute_random on the GPU against the reference's own permute_random
    (dataset.cpp:120-144): same perm, both orientations bit-exact (values
    moved, so (float) of the reference's), features / labels moved."""
    g = cg.generate_dataset(n, d, 5, 3, 1, 2, 3)
    rd = ref.dataset(n, d, 5, 3, 1, 2, 3)
    gp, perm = cg.permute_random(g, seed)
    rp_ds, rperm = rd.permute(seed)
    assert np.array_equal(perm, rperm)
    for which in (0, 1):
        a = gp.csr(which).download()
        b = rp_ds.csr(which)
        assert np.array_equal(a[0], b.row_ptr)
        assert np.array_equal(a[1], b.col_idx)
        assert np.array_equal(a[2], b.vals.astype(np.float32))
    assert np.array_equal(gp.features(), rp_ds.features().astype(np.float32))
    assert np.array_equal(gp.labels(), rp_ds.labels())
    # A permuted dataset trains like any other (smoke: finite losses).
    model = cg.init_glorot([5, 4, 3], 4, 0.5)
    t = cg.make_trainer(gp, model, cg.Strategy("1d", 1))
    t.distribute()
    assert np.all(np.isfinite(t.run_epochs(2)))


def _write_text_dataset(tmp_path, n, edges, feats, labels, header=True):
    e = tmp_path / "edges.txt"
    with open(e, "w") as fh:
        fh.write("# an edge list\n")
        if header:
            fh.write(f"% n {n}\n")
        for u, v in edges:
            fh.write(f"{u} {v}  # edge\n")
        fh.write("\n")
    f = tmp_path / "features.csv"
    with open(f, "w") as fh:
        for row in feats:
            fh.write(",".join(f"{x:.17g}" for x in row) + "\n")
    lab = tmp_path / "labels.csv"
    with open(lab, "w") as fh:
        fh.write("# vertex,label\n")
        for i, y in enumerate(labels):
            fh.write(f"{i},{y}\n")
    return str(e), str(f), str(lab)


@pytest.mark.parametrize("undirected", [False, True])
def test_load_dataset_text_formats(cg, ref, tmp_path, undirected):
    """load_dataset (dataset.cpp:293-307) against the reference's own loader:
    edge list with comments / header / duplicates, features CSV, labels."""
    rng = np.random.default_rng(5)
    n = 40
    edges = [(int(u), int(v)) for u, v in rng.integers(0, n, size=(150, 2))]
    edges += edges[:10]  # duplicates collapse (from_pairs sort + unique)
    feats = rng.standard_normal((n, 7))
    labels = rng.integers(0, 4, size=n)
    paths = _write_text_dataset(tmp_path, n, edges, feats, labels)
    g = cg.load_dataset(*paths, undirected=undirected)
    # Expected: the reference's make_dataset on from_edge_list of the same
    # pairs (the reference's own text loader misparses "% n" headers once numpy
    # is loaded in the process — iostream state — so the parse is pinned by the
    # error-path test and the C restatement of from_edge_list instead).
    import oracle
    raw = oracle.Oracle().from_edge_list(n, np.array([e[0] for e in edges]),
                                         np.array([e[1] for e in edges]), undirected)
    r = ref.dataset_make(raw, feats, labels, int(labels.max()) + 1)
    assert (g.n, g.nnz, g.num_features, g.num_classes) == (r.n, r.nnz, r.f, r.num_classes)
    for which in (0, 1):
        a, b = g.csr(which).download(), r.csr(which)
        assert np.array_equal(a[0], b.row_ptr) and np.array_equal(a[1], b.col_idx)
        assert np.array_equal(a[2], b.vals.astype(np.float32))
    assert np.array_equal(g.features(), r.features().astype(np.float32))
    assert np.array_equal(g.labels(), r.labels())


def test_load_dataset_errors(cg, tmp_path):
    n = 5
    paths = _write_text_dataset(tmp_path, n, [(0, 1), (1, 2)], np.ones((n, 2)), [0, 1, 0, 1, 0])
    with pytest.raises(cg.CagnetError, match="cannot open"):
        cg.load_dataset(str(tmp_path / "missing.txt"), paths[1], paths[2])
    bad = tmp_path / "bad_edges.txt"
    bad.write_text("% m 5\n0 1\n")
    with pytest.raises(cg.CagnetError, match="bad header at line 1"):
        cg.load_dataset(str(bad), paths[1], paths[2])
    out = tmp_path / "out_of_range.txt"
    out.write_text("% n 3\n0 4\n")
    with pytest.raises(cg.CagnetError, match="outside declared n=3"):
        cg.load_dataset(str(out), paths[1], paths[2])
    rag = tmp_path / "ragged.csv"
    rag.write_text("1,2\n3\n1,2\n1,2\n1,2\n")
    with pytest.raises(cg.CagnetError, match="ragged row at line 2"):
        cg.load_dataset(paths[0], str(rag), paths[2])
    lab = tmp_path / "labels_missing.csv"
    lab.write_text("0,1\n1,0\n")
    with pytest.raises(cg.CagnetError, match="no label for vertex 2"):
        cg.load_dataset(paths[0], paths[1], str(lab))
