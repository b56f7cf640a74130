"""Hot-path kernels through the C-ABI against the fp64 oracle: K1 SpMM,
K2 tcgen05 split-TF32 GEMM (all transposition / epilogue / split-K cases),
K3 fused log_softmax + NLL.  Tolerances are relative Frobenius, stated per
test (north star: 1e-4 for fp32 parity)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _gpu(need_gpus):
    need_gpus(1)


@pytest.fixture(scope="module")
def torch():
    import torch
    torch.cuda.init()
    return torch


def rel(a, b):
    import oracle
    return oracle.rel_frobenius(a, b)


def dev(torch, x, dtype=None):
    return torch.from_numpy(np.ascontiguousarray(x)).to(dtype=dtype).cuda()


def stream(torch):
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def padded(torch, x, ld):
    out = torch.zeros((x.shape[0], ld), dtype=torch.float32, device="cuda")
    out[:, :x.shape[1]] = torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()
    return out


@pytest.mark.parametrize("f", [1, 3, 5, 16, 24, 41, 128, 300, 602, 1100])
@pytest.mark.parametrize("acc", [0, 1])
def test_spmm_matches_oracle(cg, orc, torch, f, acc):
    n = 700
    a = orc.normalize(orc.er_generate(n, 20.0, 3))
    h = orc.random_features(n, f, 5) - 0.5
    t0 = orc.random_features(n, f, 6) if acc else np.zeros((n, f))
    want = orc.spmm(a, h, t0)
    g = cg.csr_upload(a.row_ptr, a.col_idx, n, a.vals)
    rp, ci, v = g.device_ptrs()
    for ld in (f, ((f + 3) // 4) * 4):  # unaligned (scalar) and padded (vector) layouts
        H = padded(torch, h, ld)
        T = padded(torch, t0, ld)
        cg.check(cg.lib.cagnet_spmm_csr_f32(n, n, a.nnz, rp, ci, v, H.data_ptr(), ld, f,
                                            T.data_ptr(), ld, acc, stream(torch)))
        torch.cuda.synchronize()
        got = T.cpu().numpy()[:, :f]
        assert rel(got, want) < 1e-6, (f, ld)
    # Ragged width in a padded layout: the vector path gathers the last vector of
    # every row whole, so junk (NaN) in H's padding must not reach the valid
    # columns, and T's padding columns must stay untouched.
    ld = ((f + 3) // 4) * 4 + 4
    H = padded(torch, h, ld)
    H[:, f:] = float("nan")
    T = padded(torch, t0, ld)
    T[:, f:] = 7.0
    cg.check(cg.lib.cagnet_spmm_csr_f32(n, n, a.nnz, rp, ci, v, H.data_ptr(), ld, f,
                                        T.data_ptr(), ld, acc, stream(torch)))
    torch.cuda.synchronize()
    got = T.cpu().numpy()
    assert rel(got[:, :f], want) < 1e-6, (f, "junk padding")
    assert (got[:, f:] == 7.0).all(), "spmm wrote into the padding columns"


# Fused SpMM row epilogue (the GCN layer's next dense step): raw copy, dense
# transform by a small W (both storage orders, i.e. T·W and S·Wᵀ), relu′ mask,
# relu output — against the oracle's spmm / gemm / relu compositions.
@pytest.mark.parametrize("f,fo,tw", [(16, 16, 0), (16, 41, 0), (41 - 25, 16, 1), (8, 64, 0),
                                     (24, 16, 1), (32, 24, 0), (4, 0, 0), (16, 0, 0), (13, 0, 0)])
@pytest.mark.parametrize("deg", [3.0, 40.0])
def test_spmm_fused_epilogue(cg, orc, torch, f, fo, tw, deg):
    n = 900
    a = orc.normalize(orc.er_generate(n, deg, 5))
    rng = np.random.default_rng(f * 100 + fo)
    h = rng.standard_normal((n, f))
    t = orc.spmm(a, h, np.zeros((n, f)))
    width = fo if fo else f
    if fo:
        w = rng.standard_normal((fo, f) if tw else (f, fo))
        z = orc.gemm(t, w, False, bool(tw))
    else:
        w, z = None, t
    mask = rng.standard_normal((n, width))
    g = cg.csr_upload(a.row_ptr, a.col_idx, n, a.vals)
    rp, ci, v = g.device_ptrs()
    ldh, ldz = (f + 3) // 4 * 4, (width + 3) // 4 * 4
    H = padded(torch, h, ldh)
    M = padded(torch, mask, ldz)
    W = dev(torch, w.astype(np.float32)) if fo else None
    w_sk, w_sn = ((1, f) if tw else (fo, 1)) if fo else (0, 0)
    for use_mask in (False, True):
        T = torch.zeros((n, ldz), device="cuda")
        R = torch.zeros((n, ldz), device="cuda")
        RAW = torch.zeros((n, ldh), device="cuda")
        cg.check(cg.lib.cagnet_spmm_fused_f32(
            n, n, a.nnz, rp, ci, v, H.data_ptr(), ldh, f, W.data_ptr() if fo else None, w_sk, w_sn,
            fo, M.data_ptr() if use_mask else None, ldz, T.data_ptr(), ldz, R.data_ptr(), ldz,
            RAW.data_ptr(), ldh, stream(torch)))
        torch.cuda.synchronize()
        want = z * (mask > 0) if use_mask else z
        assert rel(RAW.cpu().numpy()[:, :f], t) < 1e-6
        assert rel(T.cpu().numpy()[:, :width], want) < 2e-6
        assert rel(R.cpu().numpy()[:, :width], np.maximum(want, 0)) < 2e-6


def test_spmm_empty_rows_and_zero_nnz(cg, orc, torch):
    rp = np.array([0, 0, 2, 2, 3], np.int64)
    ci = np.array([1, 3, 0], np.int64)
    vals = np.array([0.5, -2.0, 4.0])
    g = cg.csr_upload(rp, ci, 4, vals)
    h = np.arange(12, dtype=np.float64).reshape(4, 3)
    H = padded(torch, h, 4)
    T = torch.full((4, 4), 7.0, device="cuda")
    p = g.device_ptrs()
    cg.check(cg.lib.cagnet_spmm_csr_f32(4, 4, 3, *p, H.data_ptr(), 4, 3, T.data_ptr(), 4, 0,
                                        stream(torch)))
    torch.cuda.synchronize()
    want = orc.spmm(orc.extract_block(oracle_csr(rp, ci, vals), 0, 4, 0, 4), h)
    assert np.allclose(T.cpu().numpy()[:, :3], want)
    assert np.all(T.cpu().numpy()[:, 3] == 7.0)  # never writes past f


def oracle_csr(rp, ci, vals):
    import oracle
    return oracle.CSR(len(rp) - 1, 4, rp, ci, vals)


GEMM_CASES = [
    # (m, n, k, ta, tb)
    (1000, 16, 602, 0, 0),     # T·W, Reddit layer 1
    (1000, 41, 16, 0, 0),      # T·W, output layer
    (602, 16, 5000, 1, 0),     # Hᵀ·S split-K
    (16, 41, 3000, 1, 0),
    (1000, 16, 41, 0, 1),      # S·Wᵀ
    (130, 200, 70, 0, 0),      # ragged tiles, n > 128
    (5, 3, 2, 1, 1),
    (64, 16, 0, 0, 0),         # k = 0
    (5000, 16, 16, 0, 0),      # H·W, 16-wide layer
    (5000, 21, 13, 0, 1),      # S·Wᵀ, ragged
    (12, 16, 9000, 1, 0),      # Hᵀ·S reduction
    # >= 1 M rows: the CUDA-core narrow x narrow kernels (gemm_small.cu), unaligned ld
    (1000003, 16, 16, 0, 0),
    (1000003, 21, 13, 0, 1),
    (12, 16, 1000003, 1, 0),
]


@pytest.mark.parametrize("m,n,k,ta,tb", GEMM_CASES)
@pytest.mark.parametrize("acc", [0, 1])
def test_gemm_split_tf32(cg, orc, torch, m, n, k, ta, tb, acc):
    rng = np.random.default_rng(m * 31 + n * 7 + k)
    a = rng.standard_normal((k, m) if ta else (m, k))
    b = rng.standard_normal((n, k) if tb else (k, n))
    c0 = rng.standard_normal((m, n)) if acc else np.zeros((m, n))
    want = c0 + orc.gemm(a, b, bool(ta), bool(tb))
    A = dev(torch, a.astype(np.float32))
    B = dev(torch, b.astype(np.float32))
    Cm = dev(torch, c0.astype(np.float32))
    cg.check(cg.lib.cagnet_gemm_f32(ta, tb, m, n, k, A.data_ptr(), A.shape[1], B.data_ptr(),
                                    B.shape[1], Cm.data_ptr(), n, acc, 0, None, 0, None, 0,
                                    stream(torch)))
    torch.cuda.synchronize()
    got = Cm.cpu().numpy()
    # fp32 inputs rounded from fp64: error budget ~1e-6 relative (split-TF32 ≈ fp32).
    assert rel(got, want) < 2e-6, rel(got, want)


# Padded (16 B-aligned) leading dimensions, as the trainers lay tiles out:
# these take the TMA-fed A-in-TMEM kernel (gemm_tm.cu), including the
# streamed-B split-K path of Hᵀ·S and multi-tile persistent CTAs.
TM_CASES = [
    # (m, n, k, ta, tb)
    (40000, 16, 602, 0, 0),    # T·W, Reddit layer 1 (many tiles per CTA)
    (3000, 41, 16, 0, 0),      # T·W, output layer (BN = 48)
    (3000, 16, 41, 0, 1),      # S·Wᵀ
    (1000, 64, 130, 0, 0),     # BN = 64
    (777, 32, 70, 0, 0),       # ragged M tile, BN = 32
    (602, 16, 20000, 1, 0),    # Hᵀ·S split-K, 5 M tiles
    (16, 41, 30000, 1, 0),     # Hᵀ·S, m < 128 (OOB-filled tile), BN = 48
    (300, 24, 12345, 1, 0),    # ragged K
    (16, 16, 100, 1, 0),       # K smaller than one k-block per split
    (3000, 256, 16, 0, 0),     # N > 64: column tiles (Protein's 256 classes)
    (3000, 16, 256, 0, 1),     # S·Wᵀ with K = 256
    (16, 200, 30000, 1, 0),    # Hᵀ·S with N > 64 (ragged last column tile)
    (40000, 16, 16, 0, 0),     # H·W (16 -> 16)
    (30000, 24, 16, 0, 1),     # S·Wᵀ (16 -> 24)
    (16, 16, 70000, 1, 0),     # Hᵀ·S, the 16-wide weight gradient
    (16, 16, 232965, 1, 0),    # Hᵀ·S at Reddit's K (8 K-row splits folded in fp64)
    # >= 1 M rows: the CUDA-core narrow x narrow kernels (gemm_small.cu)
    (1000003, 16, 16, 0, 0),   # H·W (16 -> 16), Amazon / Protein hidden layers (quad kernel)
    (1000003, 16, 16, 0, 1),   # S·Wᵀ (16 -> 16), quad kernel with a transposed B
    (1000003, 14, 13, 0, 0),   # quad kernel, ragged k and n
    (1000005, 3, 5, 0, 1),     # quad kernel, tiny ragged tile
    (1000003, 24, 16, 0, 1),   # S·Wᵀ (16 -> 24)
    (1000003, 16, 24, 0, 1),
    (1000003, 40, 32, 0, 0),   # two column groups per lane, ragged
    (16, 16, 1000003, 1, 0),   # Hᵀ·S, cp.async-staged reduction
    (8, 24, 1000003, 1, 0),
    (32, 32, 1000003, 1, 0),
    (3, 5, 1000003, 1, 0),     # tiny tile
]


@pytest.mark.parametrize("m,n,k,ta,tb", TM_CASES)
@pytest.mark.parametrize("acc", [0, 1])
def test_gemm_padded_ld(cg, orc, torch, m, n, k, ta, tb, acc):
    rng = np.random.default_rng(m * 13 + n * 5 + k)
    a = rng.standard_normal((k, m) if ta else (m, k))
    b = rng.standard_normal((n, k) if tb else (k, n))
    c0 = rng.standard_normal((m, n)) if acc else np.zeros((m, n))
    want = c0 + orc.gemm(a, b, bool(ta), bool(tb))
    lda = (a.shape[1] + 3) // 4 * 4
    ldb = (b.shape[1] + 3) // 4 * 4
    ldc = (n + 3) // 4 * 4
    A = padded(torch, a, lda)
    B = padded(torch, b, ldb)
    Cm = padded(torch, c0, ldc)
    cg.check(cg.lib.cagnet_gemm_f32(ta, tb, m, n, k, A.data_ptr(), lda, B.data_ptr(), ldb,
                                    Cm.data_ptr(), ldc, acc, 0, None, 0, None, 0, stream(torch)))
    torch.cuda.synchronize()
    got = Cm.cpu().numpy()[:, :n]
    assert rel(got, want) < 2e-6, rel(got, want)


@pytest.mark.parametrize("pad", [False, True])
def test_gemm_epilogues(cg, orc, torch, pad):
    rng = np.random.default_rng(4)
    m, n, k = 777, 16, 41
    a = rng.standard_normal((m, k))
    w = rng.standard_normal((k, n))
    z = orc.gemm(a, w)
    lda = 44 if pad else k
    A, W = padded(torch, a, lda), dev(torch, w.astype(np.float32))
    Z = torch.zeros((m, n), device="cuda")
    H = torch.zeros((m, n), device="cuda")
    cg.check(cg.lib.cagnet_gemm_f32(0, 0, m, n, k, A.data_ptr(), lda, W.data_ptr(), n, Z.data_ptr(), n,
                                    0, 1, None, 0, H.data_ptr(), n, stream(torch)))
    torch.cuda.synchronize()
    assert rel(Z.cpu().numpy(), z) < 2e-6
    assert rel(H.cpu().numpy(), np.maximum(z, 0)) < 2e-6
    # RELU_PRIME: C = (S · Wᵀ) ⊙ 1[aux > 0] (dense.cpp:72-92)
    s = rng.standard_normal((m, 16))
    w2 = rng.standard_normal((k, 16))
    aux = rng.standard_normal((m, k))
    want = orc.gemm(s, w2, False, True) * (aux > 0)
    ldg = 44 if pad else k
    S, W2 = dev(torch, s.astype(np.float32)), dev(torch, w2.astype(np.float32))
    AUX = padded(torch, aux, ldg)
    G = torch.zeros((m, ldg), device="cuda")
    cg.check(cg.lib.cagnet_gemm_f32(0, 1, m, k, 16, S.data_ptr(), 16, W2.data_ptr(), 16, G.data_ptr(), ldg,
                                    0, 2, AUX.data_ptr(), ldg, None, 0, stream(torch)))
    torch.cuda.synchronize()
    assert rel(G.cpu().numpy()[:, :k], want) < 2e-6
    # relu′ with accumulate (C += S Wᵀ, then the mask)
    c0 = rng.standard_normal((m, k))
    G = padded(torch, c0, ldg)
    cg.check(cg.lib.cagnet_gemm_f32(0, 1, m, k, 16, S.data_ptr(), 16, W2.data_ptr(), 16, G.data_ptr(), ldg,
                                    1, 2, AUX.data_ptr(), ldg, None, 0, stream(torch)))
    torch.cuda.synchronize()
    assert rel(G.cpu().numpy()[:, :k], (c0 + orc.gemm(s, w2, False, True)) * (aux > 0)) < 2e-6


def test_gemm_rejects_bad_shapes(cg):
    with pytest.raises(cg.InvalidArgument):
        cg.check(cg.lib.cagnet_gemm_f32(0, 0, 4, 4, 4, None, 2, None, 4, None, 4, 0, 0, None, 0,
                                        None, 0, None))


@pytest.mark.parametrize("cols,c0,c1", [(41, 0, 41), (8, 0, 8), (256, 0, 256), (41, 14, 28), (3, 2, 3)])
def test_logsoftmax_nll(cg, orc, torch, cols, c0, c1):
    rng = np.random.default_rng(cols)
    rows = 3000
    z = rng.standard_normal((rows, cols)) * 3
    labels = rng.integers(0, cols, rows)
    mask = (rng.random(rows) < 0.8).astype(np.uint8)
    total = int(mask.sum())
    logp = orc.log_softmax(z)
    loss, g = orc.nll_tile(logp[:, c0:c1], labels, mask, total, c0)
    Z = dev(torch, z.astype(np.float32))
    L = torch.zeros((rows, c1 - c0), device="cuda")
    G = torch.zeros((rows, c1 - c0), device="cuda")
    Y = dev(torch, labels.astype(np.int32))
    M = dev(torch, mask)
    loss_dev = torch.zeros(1, dtype=torch.float64, device="cuda")
    cg.check(cg.lib.cagnet_logsoftmax_nll_f32(Z.data_ptr(), rows, cols, cols, c0, c1, L.data_ptr(),
                                              c1 - c0, G.data_ptr(), c1 - c0, Y.data_ptr(),
                                              M.data_ptr(), total, loss_dev.data_ptr(), stream(torch)))
    torch.cuda.synchronize()
    assert rel(L.cpu().numpy(), logp[:, c0:c1]) < 1e-6
    assert rel(G.cpu().numpy(), g) < 1e-5
    assert abs(loss_dev.item() - loss) / max(1.0, abs(loss)) < 1e-6


@pytest.mark.parametrize("acc", [0, 1])
def test_gemm_small_epilogues(cg, orc, torch, acc):
    """Fused epilogues on the CUDA-core narrow kernels: relu(Z) side output
    (EPI_RELU) and ⊙ relu′(aux) (EPI_RELU_PRIME), with and without accumulate."""
    rng = np.random.default_rng(11 + acc)
    m, k, n = 1000003, 16, 16
    a, w = rng.standard_normal((m, k)), rng.standard_normal((k, n))
    c0 = rng.standard_normal((m, n)) if acc else np.zeros((m, n))
    z = c0 + orc.gemm(a, w)
    A, W = padded(torch, a, 16), dev(torch, w.astype(np.float32))
    Z, H = padded(torch, c0, 16), torch.zeros((m, 16), device="cuda")
    cg.check(cg.lib.cagnet_gemm_f32(0, 0, m, n, k, A.data_ptr(), 16, W.data_ptr(), n, Z.data_ptr(), 16,
                                    acc, 1, None, 0, H.data_ptr(), 16, stream(torch)))
    torch.cuda.synchronize()
    assert rel(Z.cpu().numpy(), z) < 2e-6
    assert rel(H.cpu().numpy(), np.maximum(z, 0)) < 2e-6
    aux = rng.standard_normal((m, n))
    want = (c0 + orc.gemm(a, w)) * (aux > 0)
    G = padded(torch, c0, 16)
    AUX = padded(torch, aux, 16)
    cg.check(cg.lib.cagnet_gemm_f32(0, 0, m, n, k, A.data_ptr(), 16, W.data_ptr(), n, G.data_ptr(), 16,
                                    acc, 2, AUX.data_ptr(), 16, None, 0, stream(torch)))
    torch.cuda.synchronize()
    assert rel(G.cpu().numpy(), want) < 2e-6
