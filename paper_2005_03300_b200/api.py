"""Python mirror of the reference's graph-loading, partitioning and
training-loop API (proj/include/cagnet/{dataset,gnn,dist}.hpp) over the
B200 C-ABI.  Names, argument meaning and error behaviour follow the
reference; state lives on the GPU behind the library's handles.

    data  = generate_dataset(n, degree, f, classes, sg, sf, sl)      # dataset.hpp:54-57
    model = init_glorot(dims, seed, lr)                              # gnn.hpp:41-42
    t     = make_trainer(data, model, Strategy("1d", ranks=1))       # dist.hpp:133-134
    t.distribute(); losses = t.run_epochs(5)                          # dist.hpp:87-109
    out   = run_distributed(factory, model, strat, epochs)            # dist.hpp:149-150
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import CagnetError, InvalidArgument, check, lib  # noqa: F401

KINDS = {"1d": 0, "1.5d": 1, "2d": 2, "3d": 3}
KIND_NAMES = {v: k for k, v in KINDS.items()}
GENERATORS = {"reference": 0, "skip": 1}
CATEGORIES = ("dbcast", "sbcast", "reduce", "allgather")
COUNTER_FIELDS = ("messages", "words_sent", "words_received", "payload_words", "calls")


# ---------------------------------------------------------------------------
# partitioning (dist.hpp:25-58, grid.hpp)
# ---------------------------------------------------------------------------
def ceil_div(a: int, b: int) -> int:
    if b == 0:
        raise InvalidArgument(1, "ceil_div: zero divisor")
    return (a + b - 1) // b


def block_range(n: int, parts: int, idx: int) -> tuple[int, int]:
    """dist_common.cpp:29-36 (through the C-ABI)."""
    out = np.zeros(2, np.int64)
    check(lib.cagnet_block_range(n, parts, idx, out))
    return int(out[0]), int(out[1])


def block_sizes(n: int, parts: int) -> list[int]:
    return [e - b for b, e in (block_range(n, parts, i) for i in range(parts))]


@dataclass
class Strategy:
    """dist.hpp:51-56: kind in {"1d", "1.5d", "2d", "3d"}, ranks P, 1.5D
    replication c, 2D panel block width (0 = whole panel)."""
    kind: str = "1d"
    ranks: int = 1
    repl: int = 1
    block: int = 0
    # Extension (not in the reference): narrow-first propagation Aᵀ(H W) for
    # layers with f_out < f_in (1D / 1.5D: GEMM then SpMM; 2D / 3D: the
    # row-group GEMM first, then SUMMA propagation of the f_out-wide tiles).
    reassociate: bool = False
    # Fused SpMM row epilogues (1D): 0 = off, 1 = ReLU / ⊙relu′ inside the
    # SpMM (default), 2 = also the small dense T·W / S·Wᵀ transforms.
    fuse: int = 1
    # Replay each epoch after the first as a captured CUDA graph (kernels and
    # NCCL collectives in one launch).
    graph: bool = True
    # 2D / 3D: sparse tiles broadcast once in distribute() and kept resident
    # (False: the reference's per-stage sparse broadcasts and ledger).
    resident_sparse: bool = True
    # 1D: stage panels exchanged through NVLink peer memory (CUDA IPC) instead
    # of an NCCL all-gather (same ledger; falls back when peers are unreachable).
    p2p: bool = True
    # 1D peer-memory stages: SpMM the own vertex block from the local panel
    # while the pushes fly, then the remaining columns.  Off by default: the
    # second pass costs more SpMM time (Reddit P=4: 0.074 + 0.128 ms vs
    # 0.161 ms in one pass) than the ~25 us push it hides.
    overlap: bool = False
    # 1D peer-memory stages whose per-peer slot is >= 32 MB (Amazon / Protein):
    # per-destination pushes, each peer's column block SpMM'd as its slot lands.
    # Off by default: P SpMM passes cost more than the transfer they hide
    # (Amazon P = 4: 4 x 0.55 ms vs 1.34 ms in one pass).
    pipeline: bool = False

    @property
    def kind_id(self) -> int:
        if self.kind not in KINDS:
            raise InvalidArgument(1, f"strategy: unknown kind {self.kind!r}")
        return KINDS[self.kind]


class ProcessGrid:
    """make_grid (dist_common.cpp:55-65) + ProcessGrid groups (grid.cpp)."""

    def __init__(self, strat: Strategy):
        if strat.block < 0:
            raise InvalidArgument(1, "strategy: panel block width must be non-negative")
        self.strat = strat
        out = np.zeros(4, np.int32)
        check(lib.cagnet_grid_shape(strat.kind_id, strat.ranks, strat.repl, out))
        self.kind, self.rows, self.cols, self.layers = (int(x) for x in out)
        self.ranks = strat.ranks

    def _group(self, rank: int, which: int) -> list[int]:
        buf = np.zeros(self.ranks, np.int32)
        cnt = C.c_int()
        check(lib.cagnet_grid_group(self.strat.kind_id, self.ranks, self.strat.repl, rank, which,
                                    buf, C.byref(cnt)))
        return [int(x) for x in buf[:cnt.value]]

    def world(self):
        return self._group(0, 0)

    def row_group(self, rank):
        return self._group(rank, 1)

    def col_group(self, rank):
        return self._group(rank, 2)

    def fiber_group(self, rank):
        return self._group(rank, 3)

    def tile(self, n: int, rank: int, width: int) -> tuple[int, int, int, int, int]:
        """(row_begin, row_end, col_begin, col_end, owner) of rank's H tile."""
        out = np.zeros(5, np.int64)
        check(lib.cagnet_tile_geometry(self.strat.kind_id, self.ranks, self.strat.repl, n, rank,
                                       width, out))
        return tuple(int(x) for x in out)


def make_grid(strat: Strategy) -> ProcessGrid:
    return ProcessGrid(strat)


# ---------------------------------------------------------------------------
# device CSR / datasets (dataset.hpp:31-93)
# ---------------------------------------------------------------------------
class DeviceCSR:
    """A library-owned device CSR (int64 row_ptr, int32 col_idx, fp32 values)."""

    def __init__(self, handle, owned=True):
        self.h = handle
        self.owned = owned
        shape = np.zeros(3, np.int64)
        check(lib.cagnet_csr_shape(self.h, shape))
        self.n_rows, self.n_cols, self.nnz = (int(x) for x in shape)

    def download(self):
        """(row_ptr int64, col_idx int64, values fp32) on the host."""
        rp = np.zeros(self.n_rows + 1, np.int64)
        ci = np.zeros(max(self.nnz, 1), np.int64)
        v = np.zeros(max(self.nnz, 1), np.float32)
        check(lib.cagnet_csr_download(self.h, rp.ctypes.data, ci.ctypes.data, v.ctypes.data))
        return rp, ci[:self.nnz], v[:self.nnz]

    def device_ptrs(self):
        rp, ci, v = C.c_void_p(), C.c_void_p(), C.c_void_p()
        check(lib.cagnet_csr_device_ptrs(self.h, C.byref(rp), C.byref(ci), C.byref(v)))
        return rp.value, ci.value, v.value

    def free(self):
        if self.h and self.owned:
            lib.cagnet_csr_free(self.h)
        self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _new_csr(fn, *args) -> DeviceCSR:
    out = C.c_void_p()
    check(fn(*args, C.byref(out)))
    return DeviceCSR(out)


def csr_upload(row_ptr, col_idx, n_cols, vals=None, device=0) -> DeviceCSR:
    rp = np.ascontiguousarray(row_ptr, np.int64)
    ci = np.ascontiguousarray(col_idx, np.int64)
    v = None if vals is None else np.ascontiguousarray(vals, np.float64)
    return _new_csr(lib.cagnet_csr_upload, device, len(rp) - 1, n_cols, rp, ci,
                    None if v is None else v.ctypes.data)


def generate_erdos_renyi(n, degree, seed, device=0) -> DeviceCSR:
    """csr.cpp:195-218 on the GPU, bit-exact."""
    return _new_csr(lib.cagnet_er_generate, device, n, float(degree), seed)


def add_self_loops_and_normalize(a: DeviceCSR) -> DeviceCSR:
    return _new_csr(lib.cagnet_csr_normalize, a.h)


def transpose(a: DeviceCSR) -> DeviceCSR:
    return _new_csr(lib.cagnet_csr_transpose, a.h)


def extract_block(a: DeviceCSR, r0, r1, c0, c1) -> DeviceCSR:
    return _new_csr(lib.cagnet_csr_extract_block, a.h, r0, r1, c0, c1)


class GraphDataset:
    """dataset.hpp:31-45, device resident on `device`."""

    def __init__(self, handle, device):
        self.h = handle
        self.device = device
        info = np.zeros(5, np.int64)
        check(lib.cagnet_dataset_info(self.h, info))
        self.n, self.nnz, self.num_features, self.num_classes, self._train = (int(x) for x in info)

    def save(self, path) -> None:
        """Binary dataset cache (CAGNETD1): load back with load_dataset_binary."""
        check(lib.cagnet_dataset_save(self.h, str(path).encode()))

    def train_count(self) -> int:
        return self._train

    def csr(self, which: int = 0) -> DeviceCSR:
        out = C.c_void_p()
        check(lib.cagnet_dataset_csr(self.h, which, C.byref(out)))
        return DeviceCSR(out, owned=False)

    @property
    def adj(self) -> DeviceCSR:
        return self.csr(0)

    @property
    def adj_t(self) -> DeviceCSR:
        return self.csr(1)

    def features(self) -> np.ndarray:
        out = np.zeros((self.n, self.num_features), np.float32)
        check(lib.cagnet_dataset_features(self.h, out))
        return out

    def labels(self) -> np.ndarray:
        out = np.zeros(self.n, np.int64)
        check(lib.cagnet_dataset_labels(self.h, out))
        return out

    def free(self):
        if self.h:
            lib.cagnet_dataset_free(self.h)
        self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def generate_dataset(n, degree, num_features, num_classes, seed_graph=1, seed_features=2,
                     seed_labels=3, device=0, generator="reference") -> GraphDataset:
    """generate_dataset (dataset.cpp:110-118) built on the GPU.  generator
    "reference" reproduces the reference graph bit for bit; "skip" is the
    O(nnz) ER-shaped generator for graphs too large for O(n^2) draws."""
    out = C.c_void_p()
    check(lib.cagnet_dataset_generate(device, n, float(degree), num_features, num_classes,
                                      seed_graph, seed_features, seed_labels,
                                      GENERATORS[generator], C.byref(out)))
    return GraphDataset(out, device)


def load_dataset(edges_path, features_path, labels_path, undirected=False,
                 device=0) -> GraphDataset:
    """load_dataset (dataset.hpp:96-97): the reference's text formats."""
    out = C.c_void_p()
    check(lib.cagnet_dataset_load(device, str(edges_path).encode(), str(features_path).encode(),
                                  str(labels_path).encode(), int(bool(undirected)), C.byref(out)))
    return GraphDataset(out, device)


def load_dataset_binary(path, device=0) -> GraphDataset:
    """A dataset written by GraphDataset.save (binary cache, no regeneration)."""
    out = C.c_void_p()
    check(lib.cagnet_dataset_load_binary(device, str(path).encode(), C.byref(out)))
    return GraphDataset(out, device)


def from_edge_list(n, u, v, undirected=False, device=0) -> DeviceCSR:
    """from_edge_list (csr.cpp:79-92) on the GPU: unit-valued canonical CSR."""
    u = np.ascontiguousarray(u, np.int64)
    v = np.ascontiguousarray(v, np.int64)
    if u.shape != v.shape:
        raise InvalidArgument(1, "from_edge_list: u and v differ in length")
    return _new_csr(lib.cagnet_csr_from_edge_list, device, n, len(u), u, v, int(bool(undirected)))


def permute_random(data: GraphDataset, seed: int):
    """permute_random (dataset.hpp:70-77): (permuted dataset, perm) with row i
    of the result = original vertex perm[i]; built on the dataset's GPU."""
    perm = np.zeros(max(data.n, 1), np.int64)
    out = C.c_void_p()
    check(lib.cagnet_dataset_permute_random(data.h, seed, perm.ctypes.data, C.byref(out)))
    return GraphDataset(out, data.device), perm[:data.n]


def make_dataset(raw_row_ptr, raw_col_idx, features, labels, num_classes, train_mask=None,
                 device=0) -> GraphDataset:
    """make_dataset (dataset.cpp:76-90) from a raw host CSR (canonical: sorted,
    unique columns), fp64 features, labels and optional training mask."""
    rp = np.ascontiguousarray(raw_row_ptr, np.int64)
    ci = np.ascontiguousarray(raw_col_idx, np.int64)
    x = np.ascontiguousarray(features, np.float64)
    y = np.ascontiguousarray(labels, np.int64)
    n = len(rp) - 1
    if x.shape[0] != n or y.shape[0] != n:
        raise InvalidArgument(1, f"GraphDataset: {x.shape[0]} feature rows / {y.shape[0]} labels "
                                 f"for {n} vertices")
    m = None if train_mask is None else np.ascontiguousarray(train_mask, np.uint8)
    out = C.c_void_p()
    check(lib.cagnet_dataset_make(device, n, rp, ci, x, x.shape[1], y,
                                  None if m is None else m.ctypes.data, num_classes, C.byref(out)))
    return GraphDataset(out, device)


# ---------------------------------------------------------------------------
# model (gnn.hpp:29-42)
# ---------------------------------------------------------------------------
@dataclass
class GnnModel:
    layer_dims: list
    weights: list = field(default_factory=list)
    learning_rate: float = 1.0

    def num_layers(self) -> int:
        return len(self.layer_dims)

    def flat_weights(self) -> np.ndarray:
        return np.concatenate([np.ascontiguousarray(w, np.float64).ravel() for w in self.weights])


def init_glorot(layer_dims, seed, learning_rate=1.0) -> GnnModel:
    dims = np.asarray(layer_dims, np.int64)
    if len(dims) < 2:
        raise InvalidArgument(1, f"init_glorot: need at least two layer dims, got {len(dims)}")
    total = int(sum(dims[i] * dims[i + 1] for i in range(len(dims) - 1))) if len(dims) > 1 else 0
    flat = np.zeros(max(total, 1))
    check(lib.cagnet_init_glorot(dims, len(dims), seed, flat))
    ws, off = [], 0
    for l in range(len(dims) - 1):
        k = int(dims[l] * dims[l + 1])
        ws.append(flat[off:off + k].reshape(int(dims[l]), int(dims[l + 1])).copy())
        off += k
    return GnnModel([int(d) for d in dims], ws, float(learning_rate))


# ---------------------------------------------------------------------------
# training (dist.hpp:83-150)
# ---------------------------------------------------------------------------
def kernel_launches() -> int:
    v = C.c_uint64()
    check(lib.cagnet_kernel_launches(C.byref(v)))
    return int(v.value)


def device_count() -> int:
    n = C.c_int()
    check(lib.cagnet_device_count(C.byref(n)))
    return n.value


def comm_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib.cagnet_comm_unique_id(buf))
    return buf.raw


def comm_local_id(ranks: int, device: int = 0) -> bytes:
    """Id of an in-process world: `ranks` ranks as threads of this process on
    one GPU (SimRuntime's thread-per-rank model, runtime.cpp:270-285)."""
    buf = C.create_string_buffer(128)
    check(lib.cagnet_comm_local_id(ranks, device, buf))
    return buf.raw


def comm_local_abort(nid: bytes, why: str) -> None:
    lib.cagnet_comm_local_abort(nid, why.encode())


GROUPS = {"world": 0, "row": 1, "col": 2, "fiber": 3}
DTYPES = {"f32": 0, "f64": 1, "i32": 2, "i64": 3}


class Comm:
    """RankContext (runtime.hpp:55-96): one rank's collectives over the groups
    of the strategy's process grid, on device buffers (raw pointers) and a
    CUDA stream handle; NCCL or the in-process world depending on the id."""

    def __init__(self, strat: Strategy, rank: int, comm_id: bytes | None, device: int = 0):
        out = C.c_void_p()
        check(lib.cagnet_comm_create(strat.kind_id, strat.ranks, strat.repl, rank, comm_id, device,
                                     C.byref(out)))
        self.h, self.rank = out.value, rank

    def group(self, which: str) -> list:
        members = (C.c_int * 512)()
        size = C.c_int()
        check(lib.cagnet_comm_group(self.h, GROUPS[which], members, C.byref(size)))
        return list(members[:size.value])

    def bcast(self, which, root, ptr, count, dtype="f32", category="dbcast", stream=0):
        check(lib.cagnet_comm_bcast(self.h, GROUPS[which], root, ptr, count, DTYPES[dtype],
                                    CATEGORIES.index(category), stream))

    def bcast_csr(self, which, root, row_ptr, n_rows, col_idx, vals, nnz, category="sbcast",
                  stream=0):
        check(lib.cagnet_comm_bcast_csr(self.h, GROUPS[which], root, row_ptr, n_rows, col_idx, vals,
                                        nnz, CATEGORIES.index(category), stream))

    def all_reduce(self, which, ptr, count, dtype="f32", category="reduce", stream=0):
        check(lib.cagnet_comm_allreduce(self.h, GROUPS[which], ptr, count, DTYPES[dtype],
                                        CATEGORIES.index(category), stream))

    def reduce_scatter_rows(self, which, send, recv, row_counts, cols, category="reduce", stream=0):
        check(lib.cagnet_comm_reduce_scatter_rows(self.h, GROUPS[which], send, recv,
                                                  np.asarray(row_counts, np.int64), cols,
                                                  CATEGORIES.index(category), stream))

    def all_gather_rows(self, which, send, recv, row_counts, cols, category="allgather", stream=0):
        check(lib.cagnet_comm_allgather_rows(self.h, GROUPS[which], send, recv,
                                             np.asarray(row_counts, np.int64), cols,
                                             CATEGORIES.index(category), stream))

    def ledger(self) -> dict:
        buf = np.zeros(20, np.uint64)
        check(lib.cagnet_comm_ledger(self.h, buf))
        return {c: dict(zip(COUNTER_FIELDS, (int(x) for x in buf[5 * i:5 * i + 5])))
                for i, c in enumerate(CATEGORIES)}

    def free(self):
        if self.h:
            lib.cagnet_comm_free(self.h)
        self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Trainer:
    """One rank of a partitioned trainer (dist.hpp:83-131) on the dataset's GPU."""

    def __init__(self, data: GraphDataset, model: GnnModel, strat: Strategy, rank: int = 0,
                 nccl_id: bytes | None = None):
        self.data, self.model, self.strat, self.rank = data, model, strat, rank
        dims = np.asarray(model.layer_dims, np.int64)
        w = model.flat_weights()
        out = C.c_void_p()
        nid = None if nccl_id is None else C.create_string_buffer(bytes(nccl_id), 128)
        check(lib.cagnet_trainer_create(data.h, dims, len(dims), w, model.learning_rate,
                                        strat.kind_id, strat.ranks, strat.repl, strat.block, rank,
                                        None if nid is None else C.cast(nid, C.c_void_p),
                                        C.byref(out)))
        self.h = out
        self.dims = [int(d) for d in dims]
        if strat.reassociate:
            check(lib.cagnet_trainer_set_option(self.h, b"reassociate", 1))
        check(lib.cagnet_trainer_set_option(self.h, b"fuse", int(strat.fuse)))
        check(lib.cagnet_trainer_set_option(self.h, b"graph", int(strat.graph)))
        check(lib.cagnet_trainer_set_option(self.h, b"resident_sparse",
                                            int(strat.resident_sparse)))
        check(lib.cagnet_trainer_set_option(self.h, b"p2p", int(strat.p2p)))
        check(lib.cagnet_trainer_set_option(self.h, b"overlap", int(strat.overlap)))
        check(lib.cagnet_trainer_set_option(self.h, b"pipeline", int(strat.pipeline)))

    # lifecycle -------------------------------------------------------------
    def distribute(self):
        check(lib.cagnet_trainer_distribute(self.h))

    def forward_layer(self, l: int):
        check(lib.cagnet_trainer_forward_layer(self.h, l))

    def epoch(self) -> float:
        loss = C.c_double()
        check(lib.cagnet_trainer_epoch(self.h, C.byref(loss)))
        return loss.value

    def run_epochs(self, epochs: int) -> np.ndarray:
        out = np.zeros(max(epochs, 1))
        check(lib.cagnet_trainer_run_epochs(self.h, epochs, out))
        return out[:epochs]

    def epoch_async(self):
        """Queues one epoch on the trainer's streams without waiting."""
        check(lib.cagnet_trainer_epoch_async(self.h))

    def losses(self) -> np.ndarray:
        """Every epoch loss so far (waits for queued epochs)."""
        cnt = C.c_int()
        check(lib.cagnet_trainer_losses(self.h, np.zeros(1), 0, C.byref(cnt)))
        out = np.zeros(max(cnt.value, 1))
        check(lib.cagnet_trainer_losses(self.h, out, cnt.value, C.byref(cnt)))
        return out[:cnt.value]

    def sync(self):
        check(lib.cagnet_trainer_sync(self.h))

    # geometry ----------------------------------------------------------------
    def tile(self, rank: int, width: int):
        out = np.zeros(5, np.int64)
        check(lib.cagnet_trainer_tile(self.h, rank, width, out))
        return tuple(int(x) for x in out)

    def tile_rows(self, rank):
        return self.tile(rank, 1)[:2]

    def tile_cols(self, rank, width):
        return self.tile(rank, width)[2:4]

    def tile_owner(self, rank):
        return self.tile(rank, 1)[4]

    def _tile_shape(self, width):
        r0, r1, c0, c1, _ = self.tile(self.rank, width)
        return r1 - r0, c1 - c0

    # readback ----------------------------------------------------------------
    def h_tile(self, layer: int) -> np.ndarray:
        out = np.zeros(self._tile_shape(self.dims[layer]), np.float32)
        check(lib.cagnet_trainer_h_tile(self.h, layer, out))
        return out

    def g_tile(self, idx: int) -> np.ndarray:
        out = np.zeros(self._tile_shape(self.dims[idx + 1]), np.float32)
        check(lib.cagnet_trainer_g_tile(self.h, idx, out))
        return out

    def weight(self, l: int) -> np.ndarray:
        out = np.zeros((self.dims[l], self.dims[l + 1]), np.float32)
        check(lib.cagnet_trainer_weight(self.h, l, out))
        return out

    def y(self, l: int) -> np.ndarray:
        out = np.zeros((self.dims[l], self.dims[l + 1]), np.float32)
        check(lib.cagnet_trainer_y(self.h, l, out))
        return out

    def num_parts(self) -> int:
        n = C.c_int()
        check(lib.cagnet_trainer_num_parts(self.h, C.byref(n)))
        return n.value

    def part(self, which: int, idx: int) -> DeviceCSR:
        return _new_csr(lib.cagnet_trainer_part, self.h, which, idx)

    def part_shape(self, which: int, idx: int) -> tuple:
        """(n_rows, n_cols, nnz) of a part without copying it."""
        out = np.zeros(3, np.int64)
        check(lib.cagnet_trainer_part_shape(self.h, which, idx, out))
        return tuple(int(x) for x in out)

    def ledger(self) -> dict:
        buf = np.zeros(20, np.uint64)
        check(lib.cagnet_trainer_ledger(self.h, buf))
        return {c: dict(zip(COUNTER_FIELDS, (int(x) for x in buf[5 * i:5 * i + 5])))
                for i, c in enumerate(CATEGORIES)}

    def last_epoch_ms(self) -> float:
        ms = np.zeros(8)
        check(lib.cagnet_trainer_stats(self.h, ms, np.zeros(4, np.uint64)))
        return float(ms[7])

    def set_timing(self, on: bool = True):
        check(lib.cagnet_trainer_set_timing(self.h, int(on)))

    def profile(self) -> dict:
        """{kernel name: dict(launches, ms, bytes, flops)} since the last reset."""
        n = C.c_int()
        check(lib.cagnet_trainer_profile_count(self.h, C.byref(n)))
        out = {}
        for i in range(n.value):
            name = C.create_string_buffer(64)
            v = np.zeros(4)
            check(lib.cagnet_trainer_profile_entry(self.h, i, name, 64, v))
            out[name.value.decode()] = dict(launches=int(v[0]), ms=float(v[1]), bytes=float(v[2]),
                                            flops=float(v[3]))
        return out

    def profile_reset(self):
        check(lib.cagnet_trainer_profile_reset(self.h))

    def step_host(self, x_tile: np.ndarray, labels_tile: np.ndarray) -> float:
        """One epoch from host buffers (H2D features/labels, epoch, D2H loss)."""
        loss = C.c_double()
        check(lib.cagnet_trainer_step_host(self.h, x_tile.ctypes.data, labels_tile.ctypes.data,
                                           C.byref(loss)))
        return loss.value

    def prefetch_host(self, x_tile: np.ndarray, labels_tile: np.ndarray) -> None:
        """Queue the H2D copies of a later step's inputs (returns at once; keep
        the host arrays alive and unchanged until that step ran)."""
        check(lib.cagnet_trainer_prefetch_host(self.h, x_tile.ctypes.data, labels_tile.ctypes.data))

    def step_prefetched(self) -> float:
        """One epoch on the oldest prefetched inputs; returns its loss."""
        loss = C.c_double()
        check(lib.cagnet_trainer_step_prefetched(self.h, C.byref(loss)))
        return loss.value

    def stream(self) -> int:
        s = C.c_void_p()
        check(lib.cagnet_trainer_stream(self.h, C.byref(s)))
        return s.value or 0

    def free(self):
        if self.h:
            lib.cagnet_trainer_free(self.h)
        self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def make_trainer(data, model, strat, rank=0, nccl_id=None) -> Trainer:
    return Trainer(data, model, strat, rank, nccl_id)


@dataclass
class DistOutcome:
    """dist.hpp:138-147 (fp32 device results widened to fp64 on the host)."""
    losses: np.ndarray
    h_final: np.ndarray
    y_final: list
    g_final: list
    model: GnnModel
    ledger: list  # per rank
    epoch_ms: float = 0.0  # last epoch, device time, max over ranks (GPU extension)
    prereduction_totals: np.ndarray = None  # SimRuntime gauges (3D only, runtime.cpp:287-295)
    memory_peaks: np.ndarray = None
    backend: str = "local"


def assemble_tiles(trainers, n, width, pick) -> np.ndarray:
    """Trainer::assemble_tiles (dist_common.cpp:117-145) with the bitwise
    replica check against each tile's owner."""
    out = np.zeros((n, width), np.float64)
    tiles = {t.rank: pick(t) for t in trainers}
    for t in trainers:
        r0, r1, c0, c1, owner = t.tile(t.rank, width)
        tile = tiles[t.rank]
        if tile.shape != (r1 - r0, c1 - c0):
            raise RuntimeError(f"assemble: rank {t.rank} tile is {tile.shape}")
        if owner != t.rank:
            if not np.array_equal(tile.view(np.uint32), tiles[owner].view(np.uint32)):
                raise RuntimeError(f"replica divergence: rank {t.rank} disagrees with rank {owner}")
            continue
        out[r0:r1, c0:c1] = tile
    return out


BACKENDS = {"auto": 0, "nccl": 1, "local": 2}
OPT = dict(reassociate=1, no_graph=2, no_resident_sparse=4, no_p2p=8, fuse0=16, fuse2=32,
           overlap=64, pipeline=128)


def strategy_options(strat: Strategy) -> int:
    """Strategy extension flags as the C-ABI's CAGNET_OPT_* bits."""
    opts = 0
    opts |= OPT["reassociate"] if strat.reassociate else 0
    opts |= 0 if strat.graph else OPT["no_graph"]
    opts |= 0 if strat.resident_sparse else OPT["no_resident_sparse"]
    opts |= 0 if strat.p2p else OPT["no_p2p"]
    opts |= OPT["fuse0"] if strat.fuse == 0 else OPT["fuse2"] if strat.fuse == 2 else 0
    opts |= OPT["overlap"] if strat.overlap else 0
    opts |= OPT["pipeline"] if strat.pipeline else 0
    return opts


def run_distributed(data, model: GnnModel, strat: Strategy, epochs: int,
                    comm: str = "auto") -> DistOutcome:
    """run_distributed (dist_common.cpp:205-222) through the C++ host
    (cagnet_run_distributed): one host thread per rank, each a Trainer on its
    GPU, the outcome assembled with the reference's bitwise replica checks.
    comm = "nccl": one GPU per rank (NCCL and NVLink peer memory; the dataset
    is copied to every rank's GPU); "local": every rank on the dataset's GPU
    through the in-process world; "auto": NCCL when there are >= P GPUs.
    `data` is a GraphDataset or a factory data(device) that builds it (called
    once, for device 0)."""
    if epochs <= 0:
        raise InvalidArgument(1, "run_epochs: epoch count must be positive")
    if comm not in BACKENDS:
        raise InvalidArgument(1, f"run_distributed: unknown comm backend {comm!r}")
    ProcessGrid(strat)  # validates the geometry before any GPU work
    if not isinstance(data, GraphDataset):
        data = data(0)
    dims = np.asarray(model.layer_dims, np.int64)
    out = C.c_void_p()
    check(lib.cagnet_run_distributed(data.h, dims, len(dims), model.flat_weights(),
                                     model.learning_rate, strat.kind_id, strat.ranks, strat.repl,
                                     strat.block, epochs, BACKENDS[comm], strategy_options(strat),
                                     C.byref(out)))
    h = out.value
    try:
        info = np.zeros(8, np.int64)
        check(lib.cagnet_outcome_info(h, info))
        n, L, E, P, backend, n_pre, epoch_us = (int(x) for x in info[:7])
        losses = np.zeros(E)
        check(lib.cagnet_outcome_losses(h, losses))
        h_final = np.zeros((n, int(dims[-1])))
        check(lib.cagnet_outcome_h_final(h, h_final))
        ys, gs, ws = [], [], []
        for l in range(L - 1):
            y = np.zeros((int(dims[l]), int(dims[l + 1])))
            check(lib.cagnet_outcome_y(h, l, y))
            w = np.zeros_like(y)
            check(lib.cagnet_outcome_weight(h, l, w))
            g = np.zeros((n, int(dims[l + 1])))
            check(lib.cagnet_outcome_g(h, l, g))
            ys.append(y)
            ws.append(w)
            gs.append(g)
        ledgers = []
        for r in range(P):
            buf = np.zeros(20, np.uint64)
            check(lib.cagnet_outcome_ledger(h, r, buf))
            ledgers.append({c: dict(zip(COUNTER_FIELDS, (int(x) for x in buf[5 * i:5 * i + 5])))
                            for i, c in enumerate(CATEGORIES)})
        pre = np.zeros(max(n_pre, 1), np.uint64)
        check(lib.cagnet_outcome_prereduction_totals(h, pre))
        peaks = np.zeros(max(P, 1), np.uint64)
        check(lib.cagnet_outcome_memory_peaks(h, peaks))
    finally:
        lib.cagnet_outcome_free(h)
    return DistOutcome(losses, h_final, ys, gs,
                       GnnModel([int(d) for d in dims], ws, model.learning_rate), ledgers,
                       epoch_us / 1000.0, pre[:n_pre], peaks[:P],
                       {v: k for k, v in BACKENDS.items()}[backend])


# ---------------------------------------------------------------------------
# analytic communication model (cost.hpp:27-115, cost.cpp:48-161)
# ---------------------------------------------------------------------------
COST_TERMS = {"1d": ("embedding_broadcast", "weight_gradient_reduce"),
              "1.5d": ("embedding_broadcast", "partial_reduce"),
              "2d": ("dense_panels", "sparse_panels", "weight_gradient_gather"),
              "3d": ("sparse_panels", "dense_panels")}


@dataclass
class CostParams:
    """cost.hpp:33-40: n, nnz, uniform width f, L graph convolutions, P, c."""
    n: int
    nnz: int
    f: int
    layers: int
    ranks: int = 1
    repl: int = 1

    def array(self) -> np.ndarray:
        return np.array([self.n, self.nnz, self.f, self.layers, self.ranks, self.repl], np.int64)


def ceil_lg(p: int) -> int:
    v = C.c_int64()
    check(lib.cagnet_cost_ceil_lg(p, C.byref(v)))
    return int(v.value)


def predict_cost(kind: str, params: CostParams) -> dict:
    """predict_{1d,15d,2d,3d} (cost.cpp:48-85): per-rank words / messages per
    epoch and the word terms (which sum to words)."""
    out = np.zeros(6, np.int64)
    check(lib.cagnet_cost_predict(KINDS[kind], params.array(), out))
    return {"words": int(out[0]), "messages": int(out[1]),
            "terms": dict(zip(COST_TERMS[kind], (int(x) for x in out[2:2 + int(out[5])])))}


def predict_2d_rect_layer(params: CostParams, p_rows: int, p_cols: int, alpha: float,
                          beta: float) -> float:
    v = C.c_double()
    check(lib.cagnet_cost_2d_rect_layer(params.array(), p_rows, p_cols, alpha, beta, C.byref(v)))
    return v.value


def memory_footprints(n, nnz, f, fmax, dims, repl, ranks) -> dict:
    out = np.zeros(4, np.int64)
    check(lib.cagnet_cost_memory(n, nnz, f, fmax, dims, repl, ranks, out))
    return dict(zip(("serial", "repl15d", "repl15d_single_adj", "split3d_peak"), (int(x) for x in out)))


def compare_cost(strat: Strategy, params: CostParams, ledgers: list, epochs: int) -> dict:
    """compare_cost (cost.cpp:115-161): the metered payload words per rank per
    epoch against the closed form; ledgers = per-rank dicts as Trainer.ledger()."""
    P = len(ledgers)
    buf = np.zeros(max(P, 1) * 20, np.uint64)
    for r, led in enumerate(ledgers):
        for i, c in enumerate(CATEGORIES):
            for j, fld in enumerate(COUNTER_FIELDS):
                buf[r * 20 + i * 5 + j] = led[c][fld]
    out = np.zeros(4)
    flags = np.zeros(3, np.int32)
    check(lib.cagnet_cost_compare(strat.kind_id, params.array(), buf, P, epochs, out, flags))
    return {"strategy": strat.kind, "predicted_words": int(out[0]), "extra_words": int(out[1]),
            "measured_words": float(out[2]), "ratio": float(out[3]), "exact": bool(flags[0]),
            "degenerate": bool(flags[1]), "within_band": bool(flags[2])}
