"""B200-native CAGNET full-batch GCN training step (arXiv 2005.03300).

The hot path lives in libcagnet_b200.so (CUDA for sm_100a + NCCL, C++ host
trainers) behind the C-ABI in include/cagnet_b200.h; this package is the
Python mirror of the reference's graph-loading / partitioning / training-loop
API over that C-ABI.
"""
from ._lib import LIB_PATH, CagnetError, InvalidArgument, build, check, lib  # noqa: F401
from .api import (  # noqa: F401
    CATEGORIES,
    Comm,
    CostParams,
    ceil_lg,
    compare_cost,
    memory_footprints,
    predict_2d_rect_layer,
    predict_cost,
    DeviceCSR,
    DistOutcome,
    GnnModel,
    GraphDataset,
    ProcessGrid,
    Strategy,
    Trainer,
    add_self_loops_and_normalize,
    assemble_tiles,
    block_range,
    block_sizes,
    ceil_div,
    comm_local_abort,
    comm_local_id,
    comm_unique_id,
    device_count,
    kernel_launches,
    csr_upload,
    extract_block,
    generate_dataset,
    generate_erdos_renyi,
    init_glorot,
    make_dataset,
    make_grid,
    load_dataset,
    load_dataset_binary,
    from_edge_list,
    make_trainer,
    permute_random,
    run_distributed,
    transpose,
)
