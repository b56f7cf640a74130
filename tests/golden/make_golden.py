"""Regenerates tests/golden/*.npz from the reference itself (oracle/_ref, the
unmodified reference sources compiled in place).  Run here, where
/root/reference exists:   python tests/golden/make_golden.py

The fixtures pin the CPU oracle and the GPU path on machines without the
reference tree.  Values are the reference's fp64 outputs.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402

STRATS = {  # test_dist_strategies.cpp:112-138 shapes plus the survey's config-1 shapes
    "1d_p3": ("1d", 3, 1, 0, 20, [8, 6, 4]),
    "15d_p6_c2": ("1.5d", 6, 2, 0, 20, [8, 6, 4]),
    "2d_p4": ("2d", 4, 1, 0, 18, [8, 6, 4]),
    "2d_p4_b3": ("2d", 4, 1, 3, 18, [8, 6, 4]),
    "2d_p9": ("2d", 9, 1, 0, 10, [8, 6, 4]),
    "3d_p8": ("3d", 8, 1, 0, 9, [8, 8, 4]),
    "1d_p2": ("1d", 2, 1, 0, 20, [8, 6, 4]),
    "15d_p4_c2": ("1.5d", 4, 2, 0, 20, [8, 6, 4]),
    "15d_p8_c2": ("1.5d", 8, 2, 0, 20, [8, 6, 4]),
    "1d_p8": ("1d", 8, 1, 0, 20, [8, 6, 4]),
}


def csr_dict(prefix, a, out):
    out[prefix + "_row_ptr"] = a.row_ptr
    out[prefix + "_col_idx"] = a.col_idx
    if a.vals is not None:
        out[prefix + "_vals"] = a.vals


def main():
    ref = oracle.Ref()
    g = {}
    # ER goldens (test_sparse_core.cpp:155-172) and raw arrays.
    for n, d, s in ((32, 8.0, 1), (64, 8.0, 7), (20, 4.0, 5)):
        csr_dict(f"er_{n}_{int(d)}_{s}", ref.er(n, d, s), g)

    # Pinned-loss dataset (test_gnn_reference.cpp:148-164).
    data = ref.dataset(32, 8.0, 16, 4, 1, 2, 3)
    csr_dict("ds32_adj", data.csr(0), g)
    csr_dict("ds32_adjt", data.csr(1), g)
    g["ds32_features"] = data.features()
    g["ds32_labels"] = data.labels()
    model = ref.model([16, 16, 4], 4, 0.5)
    for l, w in enumerate(model.weights()):
        g[f"ds32_w0_{l}"] = w
    res = ref.serial(data, model, 5)
    g["ds32_losses"] = res.losses
    g["ds32_h_final"] = res.h_final
    for l in range(2):
        g[f"ds32_y_{l}"] = res.y[l]
        g[f"ds32_g_{l}"] = res.g[l]
        g[f"ds32_w_{l}"] = res.w[l]
    np.savez_compressed(os.path.join(HERE, "reference_small.npz"), **g)

    # Config 1 (BASELINE configs[0]): structure and per-block nnz.
    c = {}
    d1 = ref.dataset(4096, 16.0, 128, 8, 1, 2, 3)
    a = d1.csr(0)
    c["adj_row_ptr"] = a.row_ptr
    c["adj_col_idx"] = a.col_idx.astype(np.int32)
    c["adj_vals"] = a.vals
    at = d1.csr(1)
    c["adjt_row_ptr"] = at.row_ptr
    c["adjt_col_idx"] = at.col_idx.astype(np.int32)
    c["features_head"] = d1.features()[:64]
    c["labels"] = d1.labels()
    m1 = ref.model([128, 16, 8], 4, 0.5)
    for kind, P in (("1d", 8), ("2d", 4), ("3d", 8), ("1.5d", 8)):
        t = ref.distribute(d1, m1, kind, P, 2 if kind == "1.5d" else 1, 0)
        nnz = []
        for r in range(P):
            for q in range(t.num_parts(r)):
                nnz.append([r, q, t.part(r, 0, q).nnz, t.part(r, 1, q).nnz])
        c[f"parts_{kind}_p{P}"] = np.asarray(nnz, np.int64)
    res1 = ref.serial(d1, m1, 2)
    c["serial_losses"] = res1.losses
    np.savez_compressed(os.path.join(HERE, "reference_config1.npz"), **c)

    # Distributed outcomes + ledgers on uneven partitions.
    dd = {}
    for name, (kind, P, repl, block, n, dims) in STRATS.items():
        data = ref.dataset(n, 4.0, dims[0], dims[-1], 11, 12, 13)
        model = ref.model(dims, 14, 0.5)
        out = ref.distributed(data, model, kind, P, repl, block, epochs=3)
        dd[f"{name}_losses"] = out.losses
        dd[f"{name}_h_final"] = out.h_final
        for l in range(len(dims) - 1):
            dd[f"{name}_y_{l}"] = out.y[l]
            dd[f"{name}_g_{l}"] = out.g[l]
            dd[f"{name}_w_{l}"] = out.w[l]
        dd[f"{name}_ledger"] = out.ledger
    np.savez_compressed(os.path.join(HERE, "reference_dist.npz"), **dd)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
