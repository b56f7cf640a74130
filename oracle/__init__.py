"""TEST INFRASTRUCTURE — NOT PRODUCT CODE.

CPU checkers for the CAGNET GCN hot path (arXiv 2005.03300):

* ``Oracle``  — ctypes wrapper of ``_build/liboracle.so``, the plain-C
  restatement in ``cagnet_oracle.c`` (each function cites the reference
  file:line it follows).
* ``Ref``     — ctypes wrapper of ``_ref/libcagnet_ref.so``, the UNMODIFIED
  reference sources compiled in place plus ``ref_shim.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package, and only
as the checker / the CPU baseline — never as the thing measured or shipped.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libcagnet_ref.so")
REF_TREE = "/root/reference/proj"

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")


def build(ref: bool | None = None) -> None:
    """Compile the C restatement (always) and oracle/_ref (when the reference
    tree is present — it is absent on the GPU box, which uses the prebuilt .so)."""
    targets = ["oracle"]
    if ref is None:
        ref = os.path.isdir(REF_TREE)
    if ref:
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


class CSR:
    """Host CSR triple with int64 indices and fp64 values (reference layout)."""

    def __init__(self, n_rows, n_cols, row_ptr, col_idx, vals=None):
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self.row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
        self.col_idx = np.ascontiguousarray(col_idx, dtype=np.int64)
        self.vals = None if vals is None else np.ascontiguousarray(vals, dtype=np.float64)

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = self.lib = C.CDLL(path)
        L.orc_er_generate.restype = C.c_int64
        L.orc_er_generate.argtypes = [C.c_int64, C.c_double, C.c_uint64, _i64p, C.c_void_p]
        L.orc_er_generate_mt.restype = C.c_int64
        L.orc_er_generate_mt.argtypes = [C.c_int64, C.c_double, C.c_uint64, C.c_int, _i64p,
                                         C.POINTER(C.c_void_p)]
        L.orc_free.argtypes = [C.c_void_p]
        L.orc_rng_jump.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_rng_seed.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_rng_next.restype = C.c_uint64
        L.orc_rng_next.argtypes = [C.c_void_p]
        L.orc_from_edge_list.restype = C.c_int64
        L.orc_from_edge_list.argtypes = [C.c_int64, C.c_int64, _i64p, _i64p, C.c_int, _i64p, C.c_void_p]
        L.orc_normalize.restype = C.c_int64
        L.orc_normalize.argtypes = [C.c_int64, _i64p, _i64p, _i64p, C.c_void_p, C.c_void_p]
        L.orc_transpose.argtypes = [C.c_int64, C.c_int64, _i64p, _i64p, _f64p, _i64p, _i64p, _f64p]
        L.orc_extract_block.restype = C.c_int64
        L.orc_extract_block.argtypes = [_i64p, _i64p, _f64p, C.c_int64, C.c_int64, C.c_int64,
                                        C.c_int64, _i64p, C.c_void_p, C.c_void_p]
        L.orc_spmm_add.argtypes = [C.c_int64, _i64p, _i64p, _f64p, _f64p, C.c_int64, _f64p]
        L.orc_gemm_add.argtypes = [_f64p, C.c_int64, C.c_int64, _f64p, C.c_int64, C.c_int64,
                                   _f64p, C.c_int, C.c_int]
        L.orc_log_softmax_rows.argtypes = [_f64p, C.c_int64, C.c_int64, _f64p]
        L.orc_nll_tile.restype = C.c_double
        L.orc_nll_tile.argtypes = [_f64p, C.c_int64, C.c_int64, _i64p, _u8p, C.c_int64,
                                   C.c_int64, _f64p]
        L.orc_random_features.argtypes = [C.c_int64, C.c_int64, C.c_uint64, _f64p]
        L.orc_random_labels.argtypes = [C.c_int64, C.c_int64, C.c_uint64, _i64p]
        L.orc_init_glorot.argtypes = [_i64p, C.c_int, C.c_uint64, _f64p]
        L.orc_block_range.argtypes = [C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_int64),
                                      C.POINTER(C.c_int64)]
        L.orc_train_serial.restype = C.c_int
        L.orc_train_serial.argtypes = ([C.c_int64] + [_i64p, _i64p, _f64p] * 2 +
                                       [_f64p, _i64p, _u8p, _i64p, C.c_int, C.c_double, C.c_int,
                                        _f64p, _f64p, _f64p, _f64p, _f64p])

    # --- graph construction -------------------------------------------------
    def er_generate(self, n: int, degree: float, seed: int) -> CSR:
        rp = np.zeros(n + 1, np.int64)
        nnz = self.lib.orc_er_generate(n, degree, seed, rp, None)
        ci = np.zeros(max(nnz, 1), np.int64)
        self.lib.orc_er_generate(n, degree, seed, rp, ci.ctypes.data)
        return CSR(n, n, rp, ci[:nnz], np.ones(nnz))

    def er_generate_mt(self, n: int, degree: float, seed: int, threads: int = 0) -> CSR:
        """csr.cpp:195-218 on host threads (row sub-streams by GF(2) jump-ahead),
        bit-identical to er_generate."""
        threads = threads or (os.cpu_count() or 1)
        rp = np.zeros(n + 1, np.int64)
        buf = C.c_void_p()
        nnz = self.lib.orc_er_generate_mt(n, degree, seed, threads, rp, C.byref(buf))
        if nnz < 0:
            raise ValueError("er_generate_mt failed")
        ci = np.ctypeslib.as_array(C.cast(buf, C.POINTER(C.c_int64)), shape=(max(nnz, 1),))[:nnz].copy()
        self.lib.orc_free(buf)
        return CSR(n, n, rp, ci, np.ones(nnz))

    def rng_draws(self, seed: int, skip: int, count: int) -> np.ndarray:
        """`count` raw draws of Rng(seed) after jumping `skip` draws ahead."""
        st = (C.c_uint64 * 4)()
        self.lib.orc_rng_seed(st, seed)
        self.lib.orc_rng_jump(st, skip)
        return np.array([self.lib.orc_rng_next(st) for _ in range(count)], np.uint64)

    def from_edge_list(self, n, u, v, undirected=False) -> CSR:
        u = np.ascontiguousarray(u, np.int64)
        v = np.ascontiguousarray(v, np.int64)
        rp = np.zeros(n + 1, np.int64)
        nnz = self.lib.orc_from_edge_list(n, len(u), u, v, int(undirected), rp, None)
        if nnz < 0:
            raise ValueError("from_edge_list: edge outside vertex range")
        ci = np.zeros(max(2 * len(u), 1), np.int64)
        self.lib.orc_from_edge_list(n, len(u), u, v, int(undirected), rp, ci.ctypes.data)
        return CSR(n, n, rp, ci[:nnz], np.ones(nnz))

    def normalize(self, a: CSR) -> CSR:
        n = a.n_rows
        rp = np.zeros(n + 1, np.int64)
        cap = a.nnz + n
        ci = np.zeros(cap, np.int64)
        vals = np.zeros(cap, np.float64)
        nnz = self.lib.orc_normalize(n, a.row_ptr, a.col_idx, rp, ci.ctypes.data, vals.ctypes.data)
        return CSR(n, n, rp, ci[:nnz], vals[:nnz])

    def transpose(self, a: CSR) -> CSR:
        trp = np.zeros(a.n_cols + 1, np.int64)
        tci = np.zeros(max(a.nnz, 1), np.int64)
        tv = np.zeros(max(a.nnz, 1), np.float64)
        vals = a.vals if a.vals is not None else np.ones(a.nnz)
        self.lib.orc_transpose(a.n_rows, a.n_cols, a.row_ptr, a.col_idx, vals, trp, tci, tv)
        return CSR(a.n_cols, a.n_rows, trp, tci[:a.nnz], tv[:a.nnz])

    def extract_block(self, a: CSR, r0, r1, c0, c1) -> CSR:
        rp = np.zeros(r1 - r0 + 1, np.int64)
        vals = a.vals if a.vals is not None else np.ones(max(a.nnz, 1))
        nnz = self.lib.orc_extract_block(a.row_ptr, a.col_idx, vals, r0, r1, c0, c1, rp, None, None)
        ci = np.zeros(max(nnz, 1), np.int64)
        v = np.zeros(max(nnz, 1), np.float64)
        self.lib.orc_extract_block(a.row_ptr, a.col_idx, vals, r0, r1, c0, c1, rp,
                                   ci.ctypes.data, v.ctypes.data)
        return CSR(r1 - r0, c1 - c0, rp, ci[:nnz], v[:nnz])

    def block_range(self, n: int, parts: int, idx: int):
        b, e = C.c_int64(), C.c_int64()
        self.lib.orc_block_range(n, parts, idx, C.byref(b), C.byref(e))
        return b.value, e.value

    # --- dense ----------------------------------------------------------------
    def spmm(self, a: CSR, h: np.ndarray, acc: np.ndarray | None = None) -> np.ndarray:
        h = np.ascontiguousarray(h, np.float64)
        out = np.zeros((a.n_rows, h.shape[1])) if acc is None else np.array(acc, np.float64)
        self.lib.orc_spmm_add(a.n_rows, a.row_ptr, a.col_idx, a.vals, h, h.shape[1], out)
        return out

    def gemm(self, a, b, ta=False, tb=False) -> np.ndarray:
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        m = a.shape[1] if ta else a.shape[0]
        n = b.shape[0] if tb else b.shape[1]
        out = np.zeros((m, n))
        self.lib.orc_gemm_add(a, a.shape[0], a.shape[1], b, b.shape[0], b.shape[1], out,
                              int(ta), int(tb))
        return out

    def log_softmax(self, z) -> np.ndarray:
        z = np.ascontiguousarray(z, np.float64)
        out = np.zeros_like(z)
        self.lib.orc_log_softmax_rows(z, z.shape[0], z.shape[1], out)
        return out

    def nll_tile(self, logp, labels, mask, train_total, col_begin=0):
        logp = np.ascontiguousarray(logp, np.float64)
        g = np.zeros_like(logp)
        loss = self.lib.orc_nll_tile(logp, logp.shape[0], logp.shape[1],
                                     np.ascontiguousarray(labels, np.int64),
                                     np.ascontiguousarray(mask, np.uint8), train_total,
                                     col_begin, g)
        return loss, g

    def random_features(self, n, f, seed) -> np.ndarray:
        out = np.zeros((n, f))
        self.lib.orc_random_features(n, f, seed, out)
        return out

    def random_labels(self, n, classes, seed) -> np.ndarray:
        out = np.zeros(n, np.int64)
        self.lib.orc_random_labels(n, classes, seed, out)
        return out

    def init_glorot(self, dims, seed):
        dims = np.asarray(dims, np.int64)
        total = int(sum(dims[i] * dims[i + 1] for i in range(len(dims) - 1)))
        w = np.zeros(total)
        self.lib.orc_init_glorot(dims, len(dims), seed, w)
        return split_weights(w, dims)

    # --- datasets / training ----------------------------------------------------
    def generate_dataset(self, n, degree, f, classes, sg, sf, sl):
        """dataset.cpp:110-118 restated: returns dict(adj, adj_t, features, labels, mask)."""
        raw = self.er_generate(n, degree, sg)
        adj = self.normalize(raw)
        return dict(n=n, adj=adj, adj_t=self.transpose(adj),
                    features=self.random_features(n, f, sf),
                    labels=self.random_labels(n, classes, sl),
                    mask=np.ones(n, np.uint8), num_classes=classes)

    def train_serial(self, data, dims, weights, lr, epochs):
        """gnn.cpp:122-132 restated; returns (losses, h_final, y, g, w)."""
        dims = np.asarray(dims, np.int64)
        L = len(dims)
        n = data["n"]
        w = np.concatenate([np.ascontiguousarray(x, np.float64).ravel() for x in weights])
        losses = np.zeros(epochs)
        h_final = np.zeros((n, dims[-1]))
        y = np.zeros_like(w)
        g = np.zeros(int(sum(n * dims[l] for l in range(1, L))))
        a, at = data["adj"], data["adj_t"]
        rc = self.lib.orc_train_serial(n, a.row_ptr, a.col_idx, a.vals, at.row_ptr, at.col_idx,
                                       at.vals, np.ascontiguousarray(data["features"], np.float64),
                                       data["labels"], data["mask"], dims, L, lr, epochs, w,
                                       losses, h_final, y, g)
        if rc != 0:
            raise ValueError(f"orc_train_serial failed: {rc}")
        gs, off = [], 0
        for l in range(1, L):
            gs.append(g[off:off + n * dims[l]].reshape(n, dims[l]))
            off += n * dims[l]
        return losses, h_final, split_weights(y, dims), gs, split_weights(w, dims)


def split_weights(flat, dims):
    out, off = [], 0
    for l in range(len(dims) - 1):
        k = int(dims[l] * dims[l + 1])
        out.append(flat[off:off + k].reshape(int(dims[l]), int(dims[l + 1])).copy())
        off += k
    return out


class Ref:
    """The reference implementation itself (oracle/_ref/libcagnet_ref.so)."""

    KIND = {"1d": 0, "1.5d": 1, "2d": 2, "3d": 3}

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where "
                                    "/root/reference exists")
        L = self.lib = C.CDLL(path)
        vp = C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_dataset_generate.restype = vp
        L.ref_dataset_generate.argtypes = [C.c_uint64, C.c_double] + [C.c_uint64] * 5
        L.ref_dataset_make.restype = vp
        L.ref_dataset_make.argtypes = [C.c_uint64, _i64p, _i64p, _f64p, C.c_uint64, _i64p, C.c_uint64]
        L.ref_dataset_load.restype = vp
        L.ref_dataset_load.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_int]
        L.ref_dataset_permute.restype = vp
        L.ref_dataset_permute.argtypes = [vp, C.c_uint64, _i64p]
        for fn in ("n", "nnz", "features_cols", "classes"):
            getattr(L, "ref_dataset_" + fn).restype = C.c_uint64
            getattr(L, "ref_dataset_" + fn).argtypes = [vp]
        L.ref_dataset_csr.argtypes = [vp, C.c_int, _i64p, _i64p, _f64p]
        L.ref_dataset_features.argtypes = [vp, _f64p]
        L.ref_dataset_labels.argtypes = [vp, _i64p]
        L.ref_dataset_free.argtypes = [vp]
        L.ref_er_nnz.restype = C.c_int64
        L.ref_er_nnz.argtypes = [C.c_uint64, C.c_double, C.c_uint64]
        L.ref_er_generate.argtypes = [C.c_uint64, C.c_double, C.c_uint64, _i64p, _i64p]
        L.ref_model_glorot.restype = vp
        L.ref_model_glorot.argtypes = [_u64p, C.c_int, C.c_uint64, C.c_double]
        L.ref_model_weight.argtypes = [vp, C.c_int, _f64p]
        L.ref_model_free.argtypes = [vp]
        L.ref_serial_run.restype = vp
        L.ref_serial_run.argtypes = [vp, vp, C.c_int]
        L.ref_dist_run.restype = vp
        L.ref_dist_run.argtypes = [vp, vp] + [C.c_int] * 6
        L.ref_collectives_script.argtypes = [C.c_int, C.c_int, C.c_int, _u64p, _f64p, _f64p]
        L.ref_session_create.restype = vp
        L.ref_session_create.argtypes = [vp, vp] + [C.c_int] * 5
        L.ref_session_epoch.restype = C.c_double
        L.ref_session_epoch.argtypes = [vp]
        L.ref_session_outcome.restype = vp
        L.ref_session_outcome.argtypes = [vp]
        L.ref_session_free.argtypes = [vp]
        L.ref_result_free.argtypes = [vp]
        L.ref_result_seconds.restype = C.c_double
        L.ref_result_seconds.argtypes = [vp]
        L.ref_result_losses.argtypes = [vp, _f64p]
        L.ref_result_h_final.argtypes = [vp, _f64p]
        for fn in ("y", "g", "w"):
            getattr(L, "ref_result_" + fn).argtypes = [vp, C.c_int, _f64p]
        L.ref_result_ledger.argtypes = [vp, C.c_int, C.c_int, _u64p]
        L.ref_trainer_distribute.restype = vp
        L.ref_trainer_distribute.argtypes = [vp, vp] + [C.c_int] * 4
        L.ref_trainer_free.argtypes = [vp]
        L.ref_trainer_num_parts.argtypes = [vp, C.c_int]
        L.ref_trainer_part_shape.argtypes = [vp, C.c_int, C.c_int, C.c_int, _u64p]
        L.ref_trainer_part.argtypes = [vp, C.c_int, C.c_int, C.c_int, _i64p, _i64p, _f64p]
        L.ref_trainer_tile.argtypes = [vp, C.c_int, C.c_uint64, _i64p]

    def _check(self, h):
        if not h:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return h

    def er(self, n, degree, seed) -> CSR:
        nnz = self.lib.ref_er_nnz(n, degree, seed)
        rp = np.zeros(n + 1, np.int64)
        ci = np.zeros(max(nnz, 1), np.int64)
        self.lib.ref_er_generate(n, degree, seed, rp, ci)
        return CSR(n, n, rp, ci[:nnz], np.ones(nnz))

    def dataset(self, n, degree, f, classes, sg=1, sf=2, sl=3):
        return RefDataset(self, self._check(self.lib.ref_dataset_generate(n, degree, f, classes,
                                                                          sg, sf, sl)))

    def dataset_make(self, raw: CSR, features, labels, classes):
        """make_dataset (dataset.cpp:76-90) from a raw CSR."""
        x = np.ascontiguousarray(features, np.float64)
        y = np.ascontiguousarray(labels, np.int64)
        return RefDataset(self, self._check(self.lib.ref_dataset_make(
            raw.n_rows, raw.row_ptr, raw.col_idx, x, x.shape[1], y, classes)))

    def load_dataset(self, edges, features, labels, undirected):
        return RefDataset(self, self._check(self.lib.ref_dataset_load(
            edges.encode(), features.encode(), labels.encode(), int(undirected))))

    def model(self, dims, seed, lr):
        d = np.asarray(dims, np.uint64)
        return RefModel(self, self._check(self.lib.ref_model_glorot(d, len(d), seed, lr)), dims)

    def serial(self, data, model, epochs):
        return RefResult(self, self._check(self.lib.ref_serial_run(data.h, model.h, epochs)),
                         data, model, epochs)

    def distributed(self, data, model, kind, ranks, repl=1, block=0, epochs=1, sched=0):
        h = self.lib.ref_dist_run(data.h, model.h, self.KIND[kind], ranks, repl, block, epochs,
                                  sched)
        return RefResult(self, self._check(h), data, model, epochs, ranks=ranks)

    def collectives_script(self, kind, ranks, repl=1):
        """The collective script of tests/test_gpu_comm.py on SimRuntime:
        (ledger[cat, rank, 5], reduce_scatter results, all_gather results)."""
        led = np.zeros(4 * ranks * 5, np.uint64)
        rs = np.zeros(64 * ranks)
        ag = np.zeros(64 * ranks)
        if self.lib.ref_collectives_script(self.KIND[kind], ranks, repl, led, rs, ag) != 0:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return led.reshape(4, ranks, 5), rs.reshape(ranks, 64), ag.reshape(ranks, 64)

    def session(self, data, model, kind, ranks, repl=1, block=0, sched=0):
        """run_distributed split into distribute() once + one call per epoch."""
        return RefSession(self, self._check(self.lib.ref_session_create(
            data.h, model.h, self.KIND[kind], ranks, repl, block, sched)), data, model, ranks)

    def distribute(self, data, model, kind, ranks, repl=1, block=0):
        h = self.lib.ref_trainer_distribute(data.h, model.h, self.KIND[kind], ranks, repl, block)
        return RefTrainer(self, self._check(h), ranks)


class RefDataset:
    def __init__(self, ref, h):
        self.ref, self.h = ref, h
        L = ref.lib
        self.n = L.ref_dataset_n(h)
        self.nnz = L.ref_dataset_nnz(h)
        self.f = L.ref_dataset_features_cols(h)
        self.num_classes = L.ref_dataset_classes(h)

    def csr(self, which=0) -> CSR:
        rp = np.zeros(self.n + 1, np.int64)
        ci = np.zeros(self.nnz, np.int64)
        v = np.zeros(self.nnz, np.float64)
        self.ref.lib.ref_dataset_csr(self.h, which, rp, ci, v)
        return CSR(self.n, self.n, rp, ci, v)

    def features(self):
        out = np.zeros((self.n, self.f))
        self.ref.lib.ref_dataset_features(self.h, out)
        return out

    def labels(self):
        out = np.zeros(self.n, np.int64)
        self.ref.lib.ref_dataset_labels(self.h, out)
        return out

    def permute(self, seed):
        """The reference's permute_random (dataset.cpp:120-144): (dataset, perm)."""
        perm = np.zeros(max(self.n, 1), np.int64)
        h = self.ref._check(self.ref.lib.ref_dataset_permute(self.h, seed, perm))
        return RefDataset(self.ref, h), perm[:self.n]

    def __del__(self):
        try:
            self.ref.lib.ref_dataset_free(self.h)
        except Exception:
            pass


class RefModel:
    def __init__(self, ref, h, dims):
        self.ref, self.h, self.dims = ref, h, list(dims)

    def weights(self):
        out = []
        for l in range(len(self.dims) - 1):
            w = np.zeros((self.dims[l], self.dims[l + 1]))
            self.ref.lib.ref_model_weight(self.h, l, w)
            out.append(w)
        return out

    def __del__(self):
        try:
            self.ref.lib.ref_model_free(self.h)
        except Exception:
            pass


class RefResult:
    def __init__(self, ref, h, data, model, epochs, ranks=1):
        L = ref.lib
        dims = model.dims
        n = data.n
        self.seconds = L.ref_result_seconds(h)
        self.losses = np.zeros(epochs)
        L.ref_result_losses(h, self.losses)
        self.h_final = np.zeros((n, dims[-1]))
        L.ref_result_h_final(h, self.h_final)
        self.y, self.g, self.w = [], [], []
        for l in range(len(dims) - 1):
            y = np.zeros((dims[l], dims[l + 1]))
            L.ref_result_y(h, l, y)
            self.y.append(y)
            g = np.zeros((n, dims[l + 1]))
            L.ref_result_g(h, l, g)
            self.g.append(g)
            w = np.zeros((dims[l], dims[l + 1]))
            L.ref_result_w(h, l, w)
            self.w.append(w)
        self.ledger = None
        buf = np.zeros(5, np.uint64)
        if L.ref_result_ledger(h, 0, 0, buf) == 0:
            self.ledger = np.zeros((4, ranks, 5), np.uint64)
            for c in range(4):
                for r in range(ranks):
                    L.ref_result_ledger(h, c, r, buf)
                    self.ledger[c, r] = buf
        L.ref_result_free(h)


class RefSession:
    def __init__(self, ref, h, data, model, ranks):
        self.ref, self.h, self.data, self.model, self.ranks = ref, h, data, model, ranks
        self.epochs = 0

    def epoch(self) -> float:
        sec = self.ref.lib.ref_session_epoch(self.h)
        if sec < 0:
            raise RuntimeError(self.ref.lib.ref_last_error().decode())
        self.epochs += 1
        return sec

    def outcome(self) -> "RefResult":
        h = self.ref._check(self.ref.lib.ref_session_outcome(self.h))
        return RefResult(self.ref, h, self.data, self.model, self.epochs, ranks=self.ranks)

    def __del__(self):
        try:
            if self.h:
                self.ref.lib.ref_session_free(self.h)
        except Exception:
            pass
        self.h = None


class RefTrainer:
    def __init__(self, ref, h, ranks):
        self.ref, self.h, self.ranks = ref, h, ranks

    def num_parts(self, rank):
        return self.ref.lib.ref_trainer_num_parts(self.h, rank)

    def part(self, rank, which, idx) -> CSR:
        shape = np.zeros(3, np.uint64)
        self.ref.lib.ref_trainer_part_shape(self.h, rank, which, idx, shape)
        r, c, nnz = (int(x) for x in shape)
        rp = np.zeros(r + 1, np.int64)
        ci = np.zeros(max(nnz, 1), np.int64)
        v = np.zeros(max(nnz, 1), np.float64)
        self.ref.lib.ref_trainer_part(self.h, rank, which, idx, rp, ci, v)
        return CSR(r, c, rp, ci[:nnz], v[:nnz])

    def tile(self, rank, width):
        out = np.zeros(5, np.int64)
        self.ref.lib.ref_trainer_tile(self.h, rank, width, out)
        return tuple(int(x) for x in out)

    def __del__(self):
        try:
            self.ref.lib.ref_trainer_free(self.h)
        except Exception:
            pass


def rel_frobenius(a, ref) -> float:
    """dense.cpp:190-201."""
    a = np.asarray(a, np.float64)
    ref = np.asarray(ref, np.float64)
    diff = float(np.sqrt(np.sum((a - ref) ** 2)))
    denom = float(np.sqrt(np.sum(ref * ref)))
    return diff if denom == 0.0 else diff / denom
