"""load_dataset ingest (io.cu: mapped files parsed on all host cores, pairs
sorted / deduplicated on the GPU) against the reference's own loader
(dataset.cpp:148-307 through oracle/_ref) on the reference's text formats.

Error paths are decided on the host before any device work, so they are
compared on CPU: every malformed input must raise the reference's message,
for the line the sequential reference reports first.  The reference runs in a
subprocess that does not load numpy (its iostream parse of the "% n" header
misbehaves once numpy shares the process).  Success cases (structure, values)
need the GPU.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libcagnet_ref.so")

_HELPER = r"""
import ctypes, json, sys
L = ctypes.CDLL(sys.argv[1])
L.ref_dataset_load.restype = ctypes.c_void_p
L.ref_dataset_load.argtypes = [ctypes.c_char_p] * 3 + [ctypes.c_int]
L.ref_last_error.restype = ctypes.c_char_p
for fn in ("n", "nnz", "features_cols", "classes"):
    getattr(L, "ref_dataset_" + fn).restype = ctypes.c_uint64
    getattr(L, "ref_dataset_" + fn).argtypes = [ctypes.c_void_p]
out = []
for e, f, l, u in json.loads(sys.stdin.read()):
    h = L.ref_dataset_load(e.encode(), f.encode(), l.encode(), u)
    if not h:
        out.append(["err", L.ref_last_error().decode()])
    else:
        out.append(["ok", L.ref_dataset_n(h), L.ref_dataset_nnz(h), L.ref_dataset_features_cols(h),
                    L.ref_dataset_classes(h)])
print(json.dumps(out))
"""


def ref_load_many(cases):
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built")
    r = subprocess.run([sys.executable, "-c", _HELPER, REF_SO], input=json.dumps(cases),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    return json.loads(r.stdout)


def ours(cg, e, f, l, u):
    try:
        d = cg.load_dataset(e, f, l, undirected=bool(u))
        return ["ok", d.n, d.nnz, d.num_features, d.num_classes]
    except cg.CagnetError as err:
        msg = str(err)
        return ["err", msg.split("] ", 1)[1] if msg.startswith("[cagnet code") else msg]


GOOD_F3 = "1,2\n3,4\n5,6\n"
GOOD_L3 = "0,0\n1,1\n2,0\n"

# (edges, features, labels) texts; each case is expected to FAIL in parsing.
ERROR_CASES = {
    "edge_comma": ("0,1\n", GOOD_F3, GOOD_L3),
    "edge_hex": ("0x1 2\n", GOOD_F3, GOOD_L3),
    "edge_suffix": ("1abc 2\n", GOOD_F3, GOOD_L3),
    "edge_one_field": ("% n 3\n0 1\n2\n", GOOD_F3, GOOD_L3),
    "edge_negative_wraps": ("-1 2\n", GOOD_F3, GOOD_L3),
    "edge_overflow": ("99999999999999999999 1\n", GOOD_F3, GOOD_L3),
    "edge_float": ("1.5 2\n", GOOD_F3, GOOD_L3),
    "header_key": ("% m 3\n0 1\n", GOOD_F3, GOOD_L3),
    "header_no_value": ("% n\n0 1\n", GOOD_F3, GOOD_L3),
    "header_glued": ("%n 3\n0 1\n", GOOD_F3, GOOD_L3),
    "first_error_wins": ("0 1\n% q 4\n1 2\nbad\n", GOOD_F3, GOOD_L3),
    "outside_header": ("% n 3\n0 1\n1 7\n0 9\n", GOOD_F3, GOOD_L3),
    "feat_empty_cell": ("% n 3\n0 1\n", "1,,2\n3,4,5\n6,7,8\n", GOOD_L3),
    "feat_leading_comma": ("% n 3\n0 1\n", ",1\n3,4\n5,6\n", GOOD_L3),
    "feat_overflow": ("% n 3\n0 1\n", "1e999,2\n3,4\n5,6\n", GOOD_L3),
    "feat_cr_line": ("% n 3\n0 1\n", "1,2\n\r\n3,4\n5,6\n", GOOD_L3),
    "feat_ragged": ("% n 3\n0 1\n", "1,2\n3,4,5\n6,7\n", GOOD_L3),
    "feat_ragged_then_bad": ("% n 3\n0 1\n", "1,2\n3\nx,1\n", GOOD_L3),
    "feat_empty_file": ("% n 3\n0 1\n", "\n\n", GOOD_L3),
    "feat_rows": ("% n 4\n0 1\n", GOOD_F3, GOOD_L3),
    "label_trailing_comma": ("% n 3\n0 1\n", GOOD_F3, "0,0\n1,\n2,0\n"),
    "label_no_comma": ("% n 3\n0 1\n", GOOD_F3, "0,0\n1 1\n"),
    "label_empty_vertex": ("% n 3\n0 1\n", GOOD_F3, "0,0\n,1\n"),
    "label_outside": ("% n 3\n0 1\n", GOOD_F3, "0,0\n5,1\n"),
    "label_negative_vertex": ("% n 3\n0 1\n", GOOD_F3, "0,0\n-1,1\n"),
    "label_missing": ("% n 3\n0 1\n", GOOD_F3, "0,0\n2,1\n"),
    "label_negative": ("% n 3\n0 1\n", GOOD_F3, "0,0\n1,-1\n2,0\n"),
}

GOOD_CASES = {
    "header_last_wins": ("% n 5\n% n 3\n0 1\n1 2\n", GOOD_F3, GOOD_L3),
    "comments_blank": ("# c\n0 1 # tail\n\n   \n1 2\n2 2\n", GOOD_F3, GOOD_L3),
    "signs_extra_fields": ("+0 1 junk\n1\t2\n", GOOD_F3, GOOD_L3),
    "feat_formats": ("% n 3\n0 1\n", "1.5abc,2,\n inf,-nan\n0x1p3,+4\n", GOOD_L3),
    "labels_override": ("% n 3\n0 1\n", GOOD_F3, "#h\n0,3\n1,1,9\n 2,0\n0,2\n"),
    "no_crlf_end": ("% n 3\n0 1\n1 2", "1,2\n3,4\n5,6", "0,0\n1,1\n2,0"),
}


def _write(tmp_path, name, texts):
    paths = []
    for suffix, text in zip(("edges.txt", "features.csv", "labels.csv"), texts):
        p = tmp_path / f"{name}_{suffix}"
        p.write_text(text)
        paths.append(str(p))
    return paths


def test_ingest_errors_match_reference(cg, tmp_path):
    cases, names = [], []
    for name, texts in ERROR_CASES.items():
        for u in (0, 1):
            cases.append(_write(tmp_path, name, texts) + [u])
            names.append((name, u))
    cases.append([str(tmp_path / "missing.txt")] + cases[0][1:3] + [0])
    names.append(("missing", 0))
    want = ref_load_many(cases)
    for nm, c, w in zip(names, cases, want):
        assert w[0] == "err", (nm, w)
        assert ours(cg, *c) == w, nm


def test_ingest_first_error_in_a_large_file(cg, tmp_path):
    """A 600K-line edge list split over all host threads: the reported error
    is the first bad line in file order, not the first one a thread saw."""
    rng = np.random.default_rng(3)
    uv = rng.integers(0, 5000, size=(600000, 2))
    lines = [f"{a} {b}" for a, b in uv]
    lines[450001] = "4 x"
    lines[300007] = "7,8"
    lines[599990] = "% bad"
    e = tmp_path / "big.txt"
    e.write_text("% n 5000\n" + "\n".join(lines) + "\n")
    f = tmp_path / "f.csv"
    f.write_text("1\n" * 5000)
    lab = tmp_path / "l.csv"
    lab.write_text("".join(f"{i},0\n" for i in range(5000)))
    c = [str(e), str(f), str(lab), 0]
    want = ref_load_many([c])[0]
    assert want[0] == "err" and "line 300009 " in want[1]
    assert ours(cg, *c) == want


@pytest.mark.gpu
def test_ingest_success_cases_match_reference(cg, need_gpus, tmp_path):
    need_gpus(1)
    cases, names = [], []
    for name, texts in GOOD_CASES.items():
        for u in (0, 1):
            cases.append(_write(tmp_path, name, texts) + [u])
            names.append((name, u))
    want = ref_load_many(cases)
    for nm, c, w in zip(names, cases, want):
        assert w[0] == "ok", (nm, w)
        assert ours(cg, *c) == w, nm


@pytest.mark.gpu
def test_ingest_large_graph_structure(cg, ref, need_gpus, tmp_path):
    """200K random directed / undirected edges with duplicates and self pairs:
    the GPU sort + unique gives the reference's from_edge_list CSR bit for bit."""
    need_gpus(1)
    import oracle
    rng = np.random.default_rng(11)
    n = 30000
    uv = rng.integers(0, n, size=(200000, 2))
    uv = np.concatenate([uv, uv[:5000], np.stack([np.arange(100)] * 2, 1)])
    e = tmp_path / "g.txt"
    e.write_text("\n".join(f"{a} {b}" for a, b in uv) + "\n")
    feats = rng.standard_normal((n, 3))
    f = tmp_path / "f.csv"
    f.write_text("\n".join(",".join(repr(float(x)) for x in row) for row in feats) + "\n")
    labels = rng.integers(0, 5, size=n)
    lab = tmp_path / "l.csv"
    lab.write_text("".join(f"{i},{y}\n" for i, y in enumerate(labels)))
    for undirected in (False, True):
        g = cg.load_dataset(str(e), str(f), str(lab), undirected=undirected)
        raw = oracle.Oracle().from_edge_list(n, uv[:, 0], uv[:, 1], undirected)
        r = ref.dataset_make(raw, feats, labels, int(labels.max()) + 1)
        for which in (0, 1):
            a, b = g.csr(which).download(), r.csr(which)
            assert np.array_equal(a[0], b.row_ptr) and np.array_equal(a[1], b.col_idx)
            assert np.array_equal(a[2], b.vals.astype(np.float32))
        assert np.array_equal(g.features(), feats.astype(np.float32))


def test_binary_cache_rejects_bad_files(cg, tmp_path):
    """Header checks happen on the host before any device work."""
    bad = tmp_path / "not_a_cache.bin"
    bad.write_bytes(b"hello world, not a dataset")
    with pytest.raises(cg.CagnetError, match="not a CAGNETD1 dataset cache"):
        cg.load_dataset_binary(str(bad))
    trunc = tmp_path / "truncated.bin"
    trunc.write_bytes(b"CAGNETD1" + np.array([10, 4, 3, 10, 5, 5], np.int64).tobytes() + b"\0" * 12)
    with pytest.raises(cg.CagnetError, match="truncated"):
        cg.load_dataset_binary(str(trunc))
    with pytest.raises(cg.CagnetError, match="cannot open"):
        cg.load_dataset_binary(str(tmp_path / "missing.bin"))


@pytest.mark.gpu
def test_binary_cache_roundtrip(cg, need_gpus, tmp_path):
    """save -> load_dataset_binary gives the same dataset bit for bit, and the
    same training trajectory."""
    need_gpus(1)
    d = cg.generate_dataset(3000, 20.0, 24, 6, 1, 2, 3)
    path = tmp_path / "d.cagnet"
    d.save(path)
    e = cg.load_dataset_binary(path)
    assert (e.n, e.nnz, e.num_features, e.num_classes, e.train_count()) == \
        (d.n, d.nnz, d.num_features, d.num_classes, d.train_count())
    for which in (0, 1):
        a, b = d.csr(which).download(), e.csr(which).download()
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
    assert np.array_equal(d.features(), e.features())
    assert np.array_equal(d.labels(), e.labels())
    model = cg.init_glorot([24, 8, 6], 4, 0.5)
    losses = []
    for data in (d, e):
        t = cg.make_trainer(data, model, cg.Strategy("1d", 1))
        t.distribute()
        losses.append(t.run_epochs(3))
    assert np.array_equal(losses[0], losses[1])


@pytest.mark.gpu
def test_from_edge_list_on_gpu(cg, orc, need_gpus):
    """from_edge_list golden arrays (test_sparse_core.cpp:39-55) and random
    edge lists against the C restatement, directed and undirected."""
    need_gpus(1)
    rp, ci, v = cg.from_edge_list(3, [0, 0, 2], [1, 1, 0], undirected=False).download()
    assert list(rp) == [0, 1, 1, 2] and list(ci) == [1, 0] and list(v) == [1.0, 1.0]
    rp, ci, _ = cg.from_edge_list(3, [0, 0, 2], [1, 1, 0], undirected=True).download()
    assert list(rp) == [0, 2, 3, 4] and list(ci) == [1, 2, 0, 0]
    rng = np.random.default_rng(9)
    u, w = rng.integers(0, 5000, 60000), rng.integers(0, 5000, 60000)
    for und in (False, True):
        a = cg.from_edge_list(5000, u, w, undirected=und).download()
        b = orc.from_edge_list(5000, u, w, und)
        assert np.array_equal(a[0], b.row_ptr) and np.array_equal(a[1], b.col_idx)
    with pytest.raises(cg.InvalidArgument, match=r"edge 1 = \(3, 0\) outside vertex range \[0, 3\)"):
        cg.from_edge_list(3, [0, 3], [1, 0])
