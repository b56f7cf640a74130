"""ctypes binding of libcagnet_b200.so (the C-ABI in include/cagnet_b200.h).

There is no fallback: if the shared library is missing the import fails
loudly with the command that builds it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
CSRC_DIR = os.path.join(PKG_DIR, "csrc")
LIB_PATH = os.path.join(PKG_DIR, "lib", "libcagnet_b200.so")
HEADER = os.path.join(os.path.dirname(PKG_DIR), "include", "cagnet_b200.h")

OK, EINVAL, ECUDA, ENCCL, ERUNTIME = 0, 1, 2, 3, 4


class CagnetError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[cagnet code {code}] {msg}")
        self.code = code


class InvalidArgument(CagnetError, ValueError):
    """std::invalid_argument in the reference."""


def build(jobs: int = 8) -> str:
    """Compile libcagnet_b200.so for sm_100a (nvcc cross-compiles without a GPU)."""
    subprocess.run(["make", "-s", "-C", CSRC_DIR, f"-j{jobs}"], check=True)
    return LIB_PATH


_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
vp = C.c_void_p
i32, i64, u64, f64, f32 = C.c_int, C.c_int64, C.c_uint64, C.c_double, C.c_float

# name -> argtypes (restype is int status unless listed in _RESTYPES)
SIGNATURES = {
    "cagnet_last_error": [],
    "cagnet_version": [],
    "cagnet_device_count": [C.POINTER(i32)],
    "cagnet_block_range": [i64, i32, i32, _i64p],
    "cagnet_grid_shape": [i32, i32, i32, _i32p],
    "cagnet_grid_group": [i32, i32, i32, i32, i32, _i32p, C.POINTER(i32)],
    "cagnet_tile_geometry": [i32, i32, i32, i64, i32, i64, _i64p],
    "cagnet_spmm_csr_f32": [i64, i64, i64, vp, vp, vp, vp, i64, i32, vp, i64, i32, vp],
    "cagnet_spmm_fused_f32": [i64, i64, i64, vp, vp, vp, vp, i64, i32, vp, i64, i64, i32, vp, i64,
                              vp, i64, vp, i64, vp, i64, vp],
    "cagnet_gemm_f32": [i32, i32, i64, i64, i64, vp, i64, vp, i64, vp, i64, i32, i32, vp, i64,
                        vp, i64, vp],
    "cagnet_logsoftmax_nll_f32": [vp, i64, i32, i64, i32, i32, vp, i64, vp, i64, vp, vp, i64,
                                  vp, vp],
    "cagnet_relu_f32": [vp, i64, i32, i64, vp, i64, vp],
    "cagnet_sgd_f32": [vp, vp, i64, f32, vp],
    "cagnet_csr_upload": [i32, i64, i64, _i64p, _i64p, vp, C.POINTER(vp)],
    "cagnet_csr_shape": [vp, _i64p],
    "cagnet_csr_download": [vp, vp, vp, vp],
    "cagnet_csr_device_ptrs": [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)],
    "cagnet_csr_free": [vp],
    "cagnet_er_generate": [i32, i64, f64, u64, C.POINTER(vp)],
    "cagnet_csr_normalize": [vp, C.POINTER(vp)],
    "cagnet_csr_transpose": [vp, C.POINTER(vp)],
    "cagnet_csr_extract_block": [vp, i64, i64, i64, i64, C.POINTER(vp)],
    "cagnet_dataset_generate": [i32, i64, f64, i64, i64, u64, u64, u64, i32, C.POINTER(vp)],
    "cagnet_dataset_make": [i32, i64, _i64p, _i64p, _f64p, i64, _i64p, vp, i64, C.POINTER(vp)],
    "cagnet_dataset_info": [vp, _i64p],
    "cagnet_dataset_permute_random": [vp, u64, vp, C.POINTER(vp)],
    "cagnet_dataset_save": [vp, C.c_char_p],
    "cagnet_dataset_load_binary": [i32, C.c_char_p, C.POINTER(vp)],
    "cagnet_csr_from_edge_list": [i32, i64, i64, _i64p, _i64p, i32, C.POINTER(vp)],
    "cagnet_dataset_load": [i32, C.c_char_p, C.c_char_p, C.c_char_p, i32, C.POINTER(vp)],
    "cagnet_dataset_csr": [vp, i32, C.POINTER(vp)],
    "cagnet_dataset_features": [vp, _f32p],
    "cagnet_dataset_labels": [vp, _i64p],
    "cagnet_dataset_free": [vp],
    "cagnet_init_glorot": [_i64p, i32, u64, _f64p],
    "cagnet_comm_unique_id": [C.c_char_p],
    "cagnet_comm_local_id": [i32, i32, C.c_char_p],
    "cagnet_comm_local_abort": [C.c_char_p, C.c_char_p],
    "cagnet_trainer_create": [vp, _i64p, i32, _f64p, f64, i32, i32, i32, i32, i32, vp,
                              C.POINTER(vp)],
    "cagnet_trainer_distribute": [vp],
    "cagnet_trainer_forward_layer": [vp, i32],
    "cagnet_trainer_epoch": [vp, C.POINTER(f64)],
    "cagnet_trainer_run_epochs": [vp, i32, _f64p],
    "cagnet_trainer_sync": [vp],
    "cagnet_trainer_epoch_async": [vp],
    "cagnet_trainer_losses": [vp, _f64p, i32, C.POINTER(i32)],
    "cagnet_trainer_tile": [vp, i32, i64, _i64p],
    "cagnet_trainer_h_tile": [vp, i32, _f32p],
    "cagnet_trainer_g_tile": [vp, i32, _f32p],
    "cagnet_trainer_weight": [vp, i32, _f32p],
    "cagnet_trainer_y": [vp, i32, _f32p],
    "cagnet_trainer_num_parts": [vp, C.POINTER(i32)],
    "cagnet_trainer_part": [vp, i32, i32, C.POINTER(vp)],
    "cagnet_trainer_part_shape": [vp, i32, i32, _i64p],
    "cagnet_trainer_stats": [vp, _f64p, _u64p],
    "cagnet_trainer_ledger": [vp, _u64p],
    "cagnet_trainer_set_timing": [vp, i32],
    "cagnet_trainer_stream": [vp, C.POINTER(vp)],
    "cagnet_trainer_set_option": [vp, C.c_char_p, i64],
    "cagnet_trainer_profile_count": [vp, C.POINTER(i32)],
    "cagnet_trainer_profile_entry": [vp, i32, C.c_char_p, i32, _f64p],
    "cagnet_trainer_profile_reset": [vp],
    "cagnet_trainer_step_host": [vp, vp, vp, C.POINTER(f64)],
    "cagnet_trainer_prefetch_host": [vp, vp, vp],
    "cagnet_trainer_step_prefetched": [vp, C.POINTER(f64)],
    "cagnet_kernel_launches": [C.POINTER(u64)],
    "cagnet_comm_create": [i32, i32, i32, i32, C.c_char_p, i32, C.POINTER(vp)],
    "cagnet_comm_group": [vp, i32, C.POINTER(i32), C.POINTER(i32)],
    "cagnet_comm_bcast": [vp, i32, i32, vp, i64, i32, i32, vp],
    "cagnet_comm_bcast_csr": [vp, i32, i32, vp, i64, vp, vp, i64, i32, vp],
    "cagnet_comm_allreduce": [vp, i32, vp, i64, i32, i32, vp],
    "cagnet_comm_reduce_scatter_rows": [vp, i32, vp, vp, _i64p, i64, i32, vp],
    "cagnet_comm_allgather_rows": [vp, i32, vp, vp, _i64p, i64, i32, vp],
    "cagnet_comm_ledger": [vp, _u64p],
    "cagnet_comm_free": [vp],
    "cagnet_cost_predict": [i32, _i64p, _i64p],
    "cagnet_cost_ceil_lg": [i64, C.POINTER(i64)],
    "cagnet_cost_2d_rect_layer": [_i64p, i64, i64, f64, f64, C.POINTER(f64)],
    "cagnet_cost_memory": [i64, i64, i64, i64, i64, i64, i64, _i64p],
    "cagnet_cost_compare": [i32, _i64p, _u64p, i32, i32, _f64p, _i32p],
    "cagnet_run_distributed": [vp, _i64p, i32, _f64p, f64, i32, i32, i32, i32, i32, i32, C.c_uint32,
                               C.POINTER(vp)],
    "cagnet_outcome_info": [vp, _i64p],
    "cagnet_outcome_losses": [vp, _f64p],
    "cagnet_outcome_h_final": [vp, _f64p],
    "cagnet_outcome_g": [vp, i32, _f64p],
    "cagnet_outcome_y": [vp, i32, _f64p],
    "cagnet_outcome_weight": [vp, i32, _f64p],
    "cagnet_outcome_ledger": [vp, i32, _u64p],
    "cagnet_outcome_prereduction_totals": [vp, _u64p],
    "cagnet_outcome_memory_peaks": [vp, _u64p],
    "cagnet_outcome_free": [vp],
    "cagnet_trainer_free": [vp],
}
_RESTYPES = {"cagnet_last_error": C.c_char_p, "cagnet_version": i32}


def _preload_nccl() -> None:
    """Bind libnccl.so.2 to the NCCL that PyTorch ships (2.28) before our
    library pulls in the older system copy, so both share one NCCL."""
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia.nccl")
        for base in (spec.submodule_search_locations or []) if spec else []:
            path = os.path.join(base, "lib", "libnccl.so.2")
            if os.path.exists(path):
                C.CDLL(path, mode=C.RTLD_GLOBAL)
                return
    except Exception:
        pass


def _load() -> C.CDLL:
    _preload_nccl()
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA extension first "
            f"(python -c 'import __graft_entry__ as g; g.build()' or make -C {CSRC_DIR})")
    lib = C.CDLL(LIB_PATH)
    for name, argtypes in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = _RESTYPES.get(name, C.c_int)
    return lib


lib = _load()


def check(code: int) -> None:
    if code == OK:
        return
    msg = lib.cagnet_last_error().decode(errors="replace")
    if code == EINVAL:
        raise InvalidArgument(code, msg)
    raise CagnetError(code, msg)


def header_symbols(path: str = HEADER) -> list[str]:
    """Names of every function the public header declares."""
    import re
    text = open(path).read()
    return sorted(set(re.findall(r"^\s*(?:CAGNET_API\s+)?(?:const\s+)?\w+\*?\s+\*?(cagnet_\w+)\s*\(", text,
                                 flags=re.M)))
