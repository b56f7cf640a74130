"""Run-to-run determinism of the multi-rank paths on the Reddit-shaped graph.

Every kernel and collective of the product is deterministic (fixed fold
orders, no float atomics), so repeated runs of the same strategy must agree
BITWISE; any difference is a race.  Round 2 found one this way: a lazily
allocated tile (the kept T = AᵀH of a widening layer) was zeroed by a
legacy-stream cudaMemset that does not order against the trainers'
non-blocking streams, so the zeroing could land after the first epoch's
writes (about half of the 2D / 3D in-process runs gave a wrong last-layer
weight gradient).  Also: the packed SpMM stream (SpmmPacked) against the
interleaved one in a separate process (CAGNET_SPMM_PACK=0)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N, E, DIMS = 232965, 114848857, [602, 16, 16, 41]


@pytest.fixture(scope="module")
def reddit(cg):
    d = cg.generate_dataset(N, E / N, DIMS[0], DIMS[-1], 1, 2, 3, device=0)
    yield d
    d.free()


def outcome_arrays(out):
    arrs = {"h_final": out.h_final, "losses": np.asarray(out.losses)}
    for l in range(len(DIMS) - 1):
        arrs[f"y{l}"] = out.y_final[l]
        arrs[f"w{l}"] = out.model.weights[l]
    return arrs


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("kind,P,graph", [("2d", 4, True), ("2d", 4, False), ("3d", 8, True)])
def test_in_process_runs_are_bitwise_repeatable(cg, reddit, need_gpus, kind, P, graph):
    need_gpus(1)
    model = cg.init_glorot(DIMS, 4, 0.5)
    single = outcome_arrays(cg.run_distributed(reddit, model, cg.Strategy("1d", 1, reassociate=True), 2))
    first = None
    for rep in range(6):
        out = outcome_arrays(cg.run_distributed(
            reddit, model, cg.Strategy(kind, P, 1, reassociate=True, graph=graph), 2, comm="local"))
        if first is None:
            first = out
            errs = {k: rel(out[k], single[k]) for k in out}
            assert max(errs.values()) < 1e-4, errs
            continue
        for k in out:
            assert np.array_equal(out[k], first[k]), (rep, k, float(np.max(np.abs(out[k] - first[k]))))


PACK_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[2])
import paper_2005_03300_b200 as cg
N, E, DIMS = 232965, 114848857, [602, 16, 16, 41]
d = cg.generate_dataset(N, E / N, DIMS[0], DIMS[-1], 1, 2, 3, device=0)
out = cg.run_distributed(d, cg.init_glorot(DIMS, 4, 0.5), cg.Strategy("1d", 1, reassociate=True), 3)
arrs = {"h_final": out.h_final, "losses": np.asarray(out.losses)}
for l in range(len(DIMS) - 1):
    arrs[f"y{l}"] = out.y_final[l]; arrs[f"w{l}"] = out.model.weights[l]
np.savez(sys.argv[1], **arrs)
"""


def test_packed_stream_matches_interleaved(tmp_path, need_gpus):
    """The packed stream (4 B per nonzero, value rebuilt as s_row * rsqrt(d_col))
    against the interleaved {col, value} stream on the 1D Reddit epoch: the
    values differ by a few ulp, every output within 1e-5."""
    need_gpus(1)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for pack in ("1", "0"):
        path = str(tmp_path / f"pack{pack}.npz")
        env = dict(os.environ, CAGNET_SPMM_PACK=pack)
        subprocess.run([sys.executable, "-c", PACK_SCRIPT, path, root], check=True, env=env, timeout=600)
        res[pack] = np.load(path)
    errs = {k: rel(res["1"][k], res["0"][k]) for k in res["0"].files}
    assert max(errs.values()) < 1e-5, errs
    assert any(v > 0 for v in errs.values()), "the packed stream did not engage"


TAMPER_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[3])
import paper_2005_03300_b200 as cg
d = cg.load_dataset_binary(sys.argv[1], device=0)
dims = [16, 16, 16, 4]
out = cg.run_distributed(d, cg.init_glorot(dims, 4, 0.5), cg.Strategy("1d", 1, reassociate=True), 3)
np.savez(sys.argv[2], h=out.h_final, y0=out.y_final[0], y1=out.y_final[1], losses=np.asarray(out.losses))
"""


def test_packed_stream_falls_back_off_normalized_values(cg, tmp_path, need_gpus):
    """A dataset whose adjacency values are not 1/sqrt(d_r d_c) (a binary cache
    with every value scaled by 1.01, A and Aᵀ alike) fails the packed stream's
    check at distribute(): the SpMMs keep the interleaved stream, so the run
    is bitwise the CAGNET_SPMM_PACK=0 run — while on the untampered cache the
    packed stream engages (results differ in the last bits)."""
    need_gpus(1)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    d = cg.generate_dataset(3000, 24.0, 16, 4, 1, 2, 3, device=0)
    clean = str(tmp_path / "clean.bin")
    d.save(clean)
    n, nnz, nnz_t = d.n, None, None
    raw = bytearray(open(clean, "rb").read())
    hdr = np.frombuffer(bytes(raw[8:8 + 48]), dtype=np.int64)
    assert hdr[0] == n
    nnz, nnz_t = int(hdr[4]), int(hdr[5])
    off = 8 + 48
    for m in (nnz, nnz_t):
        off += (n + 1) * 8 + m * 4
        vals = np.frombuffer(bytes(raw[off:off + m * 4]), dtype=np.float32) * np.float32(1.01)
        raw[off:off + m * 4] = vals.astype(np.float32).tobytes()
        off += m * 4
    tampered = str(tmp_path / "tampered.bin")
    open(tampered, "wb").write(bytes(raw))
    res = {}
    for name, path in (("clean", clean), ("tampered", tampered)):
        for pack in ("1", "0"):
            outp = str(tmp_path / f"{name}{pack}.npz")
            subprocess.run([sys.executable, "-c", TAMPER_SCRIPT, path, outp, root], check=True,
                           env=dict(os.environ, CAGNET_SPMM_PACK=pack), timeout=300)
            res[name + pack] = np.load(outp)
    for k in res["tampered0"].files:
        assert np.array_equal(res["tampered1"][k], res["tampered0"][k]), k
    assert any(not np.array_equal(res["clean1"][k], res["clean0"][k]) for k in res["clean0"].files)
    errs = {k: rel(res["clean1"][k], res["clean0"][k]) for k in res["clean0"].files}
    assert max(errs.values()) < 1e-5, errs
