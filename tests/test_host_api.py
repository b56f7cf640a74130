"""Host-side checks that need no GPU: the C-ABI library loads and exports
every symbol the public header declares, and the partition geometry
(block ranges, grids, groups, tiles) equals the reference's."""
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_library_exports_header(cg):
    from paper_2005_03300_b200._lib import LIB_PATH, header_symbols, lib
    syms = header_symbols()
    assert len(syms) >= 40
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert os.path.basename(LIB_PATH) == "libcagnet_b200.so"
    assert lib.cagnet_version() == 1


def test_sass_is_sm100a_with_tcgen05(cg):
    import shutil
    import subprocess
    from paper_2005_03300_b200._lib import LIB_PATH
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "-lelf", LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass, "tcgen05.mma (kind::tf32) missing from the GEMM"
    assert "LDTM" in sass, "tcgen05.ld missing from the GEMM epilogue"


def test_block_range_golden(cg):
    assert cg.block_sizes(10, 4) == [3, 3, 3, 1]
    assert cg.block_sizes(3, 4) == [1, 1, 1, 0]
    assert cg.block_sizes(12, 3) == [4, 4, 4]
    for n in (1, 7, 12, 13):
        for parts in (1, 2, 3, 5):
            prev = 0
            for i in range(parts):
                b, e = cg.block_range(n, parts, i)
                assert b == prev
                prev = e
            assert prev == n
    with pytest.raises(cg.InvalidArgument):
        cg.block_range(10, 4, 4)
    with pytest.raises(cg.InvalidArgument):
        cg.block_range(10, 0, 0)
    assert cg.ceil_div(10, 4) == 3 and cg.ceil_div(0, 4) == 0


# test_dist.cpp:124-165
def test_grid_groups_golden(cg):
    g15 = cg.ProcessGrid(cg.Strategy("1.5d", 8, 2))
    assert (g15.rows, g15.cols) == (4, 2)
    assert g15.col_group(4) == [0, 2, 4, 6]
    assert g15.row_group(4) == [4, 5]
    g2 = cg.ProcessGrid(cg.Strategy("2d", 9))
    assert g2.rows == 3 and g2.row_group(4) == [3, 4, 5] and g2.col_group(4) == [1, 4, 7]
    g3 = cg.ProcessGrid(cg.Strategy("3d", 8))
    assert g3.layers == 2
    assert g3.fiber_group(1) == [1, 5] and g3.row_group(1) == [0, 1] and g3.col_group(1) == [1, 3]
    assert cg.ProcessGrid(cg.Strategy("1d", 3)).world() == [0, 1, 2]


@pytest.mark.parametrize("bad", [("2d", 6, 1, 0), ("3d", 9, 1, 0), ("1.5d", 6, 4, 0),
                                 ("1d", 0, 1, 0), ("1d", 2, 1, -1)])
def test_make_grid_validation(cg, bad):
    with pytest.raises(cg.InvalidArgument):
        cg.make_grid(cg.Strategy(*bad))


def test_tile_geometry_matches_reference(cg, ref):
    # Every strategy shape of the reference tests, on uneven n.
    data = ref.dataset(13, 3.0, 8, 4, 1, 2, 3)
    model = ref.model([8, 6, 4], 4, 0.5)
    for kind, P, c in (("1d", 3, 1), ("1.5d", 8, 2), ("1.5d", 6, 2), ("2d", 4, 1), ("2d", 9, 1),
                       ("3d", 8, 1), ("1.5d", 2, 2)):
        t = ref.distribute(data, model, kind, P, c, 0)
        grid = cg.ProcessGrid(cg.Strategy(kind, P, c))
        owned = 0
        for r in range(P):
            for width in (6, 4, 1):
                assert grid.tile(13, r, width) == t.tile(r, width), (kind, P, r, width)
            r0, r1, c0, c1, owner = grid.tile(13, r, 6)
            if owner == r:
                owned += (r1 - r0) * (c1 - c0)
        assert owned == 13 * 6


def test_glorot_matches_oracle(cg, orc):
    m = cg.init_glorot([602, 16, 16, 41], 4, 0.5)
    w = orc.init_glorot([602, 16, 16, 41], 4)
    for a, b in zip(m.weights, w):
        assert np.array_equal(a, b)
    with pytest.raises(cg.InvalidArgument):
        cg.init_glorot([5], 1)
    with pytest.raises(cg.InvalidArgument):
        cg.init_glorot([5, 0, 2], 1)


def test_product_has_no_oracle_dependency():
    """The shipped package must never route through the CPU checker."""
    pkg = os.path.join(os.path.dirname(os.path.dirname(__file__)), "paper_2005_03300_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".hpp", ".cpp", ".h")):
                text = open(os.path.join(root, f)).read()
                assert "import oracle" not in text and "cagnet_oracle" not in text, f
