"""End-to-end GCN training on the GPU against the serial fp64 oracle — the
verify_against_serial recipe (harness.cpp:118-166) at the north star's fp32
tolerance: h_final, every y_l, g_l, w_l within 1e-4 relative Frobenius and
the loss |Δ|/max(1,|loss|) <= 1e-4 per epoch (test_dist_strategies.cpp:63-66)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
TOL = 1e-4


@pytest.fixture(autouse=True)
def _gpu(need_gpus):
    need_gpus(1)


def max_rel_error(out, ref_losses, ref_h, ref_y, ref_g, ref_w):
    import oracle
    worst = oracle.rel_frobenius(out["h_final"], ref_h)
    for l in range(len(ref_y)):
        worst = max(worst, oracle.rel_frobenius(out["y"][l], ref_y[l]))
        worst = max(worst, oracle.rel_frobenius(out["g"][l], ref_g[l]))
        worst = max(worst, oracle.rel_frobenius(out["w"][l], ref_w[l]))
    for a, b in zip(out["losses"], ref_losses):
        worst = max(worst, abs(a - b) / max(1.0, abs(b)))
    return worst


def run_single(cg, data, model, strat, epochs):
    t = cg.make_trainer(data, model, strat)
    t.distribute()
    losses = t.run_epochs(epochs)
    L = len(model.layer_dims)
    return dict(losses=losses, h_final=t.h_tile(L - 1).astype(np.float64),
                y=[t.y(l).astype(np.float64) for l in range(L - 1)],
                g=[t.g_tile(l).astype(np.float64) for l in range(L - 1)],
                w=[t.weight(l).astype(np.float64) for l in range(L - 1)], trainer=t)


@pytest.mark.parametrize("strat", [("1d", 1, 1, 0), ("1.5d", 1, 1, 0), ("2d", 1, 1, 0),
                                   ("2d", 1, 1, 3), ("3d", 1, 1, 0)])
def test_single_rank_matches_serial(cg, orc, strat):
    dims = [12, 10, 7, 5]
    data = cg.generate_dataset(64, 8.0, dims[0], dims[-1], 7, 8, 9)
    model = cg.init_glorot(dims, 3, 0.25)
    od = orc.generate_dataset(64, 8.0, dims[0], dims[-1], 7, 8, 9)
    losses, h, y, g, w = orc.train_serial(od, dims, model.weights, 0.25, 3)
    out = run_single(cg, data, model, cg.Strategy(*strat), 3)
    err = max_rel_error(out, losses, h, y, g, w)
    assert err < TOL, err
    led = out["trainer"].ledger()
    assert all(v == 0 for c in led.values() for v in c.values())  # P = 1 meters nothing


@pytest.mark.parametrize("kind", ["1d", "1.5d", "2d", "3d"])
@pytest.mark.parametrize("fuse", [0, 1, 2])
@pytest.mark.parametrize("dims", [[40, 12, 7, 5], [40, 16, 16, 24], [20, 16, 41]])
def test_reassociated_matches_serial(cg, orc, kind, fuse, dims):
    """Narrow-first propagation Aᵀ(H W): same GCN, f_out-wide panels; with and
    without the fused SpMM row epilogues (ReLU, T·W, S·Wᵀ ⊙ relu′, relu′);
    Reddit-shaped widths (narrow, equal and widening output layers)."""
    data = cg.generate_dataset(96, 9.0, dims[0], dims[-1], 7, 8, 9)
    model = cg.init_glorot(dims, 3, 0.25)
    od = orc.generate_dataset(96, 9.0, dims[0], dims[-1], 7, 8, 9)
    losses, h, y, g, w = orc.train_serial(od, dims, model.weights, 0.25, 3)
    out = run_single(cg, data, model, cg.Strategy(kind, 1, 1, 0, reassociate=True, fuse=fuse), 3)
    assert max_rel_error(out, losses, h, y, g, w) < TOL


@pytest.mark.parametrize("kind", ["1d", "2d", "3d"])
def test_graph_replay_matches_eager(cg, kind):
    """Epochs replayed from the captured CUDA graph are bit-identical to the
    eager epochs (same kernels, same order); losses land at the device-side
    slot, so every replay appends its own loss."""
    dims = [40, 16, 16, 24]
    data = cg.generate_dataset(96, 9.0, dims[0], dims[-1], 7, 8, 9)
    model = cg.init_glorot(dims, 3, 0.25)
    outs = []
    for graph in (False, True):
        t = cg.make_trainer(data, model, cg.Strategy(kind, 1, 1, 0, reassociate=True,
                                                     graph=graph))
        t.distribute()
        losses = t.run_epochs(6)
        more = [t.epoch() for _ in range(3)]
        outs.append((np.concatenate([losses, more]), [t.weight(l) for l in range(len(dims) - 1)],
                     t.h_tile(len(dims) - 1)))
    (l0, w0, h0), (l1, w1, h1) = outs
    assert len(l1) == 9 and len(set(np.round(l1, 12))) > 1
    assert np.array_equal(l0, l1)
    assert all(np.array_equal(a, b) for a, b in zip(w0, w1))
    assert np.array_equal(h0, h1)


def test_pinned_loss_trace_fp32(cg):
    expected = [1.4676915537761182, 1.3547714828994135, 1.3527671034478277,
                1.3514914086563463, 1.3507757616337233]
    data = cg.generate_dataset(32, 8.0, 16, 4, 1, 2, 3)
    assert data.nnz == 281
    model = cg.init_glorot([16, 16, 4], 4, 0.5)
    t = cg.make_trainer(data, model, cg.Strategy("1d", 1))
    t.distribute()
    losses = t.run_epochs(5)
    for a, b in zip(losses, expected):
        assert abs(a - b) / max(1.0, abs(b)) < TOL
    assert losses[-1] < losses[0]


def test_config1_matches_serial(cg, orc):
    """BASELINE configs[0]: ER n=4096 d=16, dims {128,16,8}, 1D P=1."""
    dims = [128, 16, 8]
    data = cg.generate_dataset(4096, 16.0, 128, 8, 1, 2, 3)
    model = cg.init_glorot(dims, 4, 0.5)
    od = orc.generate_dataset(4096, 16.0, 128, 8, 1, 2, 3)
    losses, h, y, g, w = orc.train_serial(od, dims, model.weights, 0.5, 3)
    out = run_single(cg, data, model, cg.Strategy("1d", 1), 3)
    assert max_rel_error(out, losses, h, y, g, w) < TOL
    c = np.load(os.path.join(GOLD, "reference_config1.npz"))
    assert np.allclose(out["losses"][:2], c["serial_losses"], rtol=TOL, atol=0)


def test_forward_layer_alone(cg, orc):
    dims = [9, 6, 4]
    data = cg.generate_dataset(50, 5.0, 9, 4, 1, 2, 3)
    model = cg.init_glorot(dims, 5, 0.5)
    t = cg.make_trainer(data, model, cg.Strategy("1d", 1))
    t.distribute()
    t.forward_layer(1)
    od = orc.generate_dataset(50, 5.0, 9, 4, 1, 2, 3)
    z = orc.gemm(orc.spmm(od["adj_t"], od["features"]), model.weights[0])
    import oracle
    assert oracle.rel_frobenius(t.h_tile(1), np.maximum(z, 0)) < 1e-5
    with pytest.raises(cg.InvalidArgument):
        t.forward_layer(3)


def test_trainer_rejects_bad_models(cg):
    data = cg.generate_dataset(10, 3.0, 8, 4, 1, 2, 3)
    with pytest.raises(cg.InvalidArgument):
        cg.make_trainer(data, cg.init_glorot([7, 6, 4], 4), cg.Strategy("1d", 1))
    with pytest.raises(cg.InvalidArgument):
        cg.make_trainer(data, cg.init_glorot([8, 6, 5], 4), cg.Strategy("1d", 1))
    with pytest.raises(cg.InvalidArgument):
        cg.make_trainer(data, cg.init_glorot([8, 6, 4], 4), cg.Strategy("2d", 2))


def test_make_dataset_from_host_arrays(cg, orc):
    raw = orc.er_generate(80, 6.0, 2)
    x = orc.random_features(80, 5, 3)
    y = orc.random_labels(80, 3, 4)
    mask = (np.arange(80) % 3 != 0).astype(np.uint8)
    data = cg.make_dataset(raw.row_ptr, raw.col_idx, x, y, 3, train_mask=mask)
    assert data.train_count() == int(mask.sum())
    model = cg.init_glorot([5, 4, 3], 9, 0.5)
    adj = orc.normalize(raw)
    od = dict(n=80, adj=adj, adj_t=orc.transpose(adj), features=x, labels=y, mask=mask)
    losses, h, yy, g, w = orc.train_serial(od, [5, 4, 3], model.weights, 0.5, 2)
    out = run_single(cg, data, model, cg.Strategy("1d", 1), 2)
    assert max_rel_error(out, losses, h, yy, g, w) < TOL


# ---- multi-GPU: every strategy vs the reference's own distributed outcome -----
DIST = {  # name -> (kind, P, repl, block, n, dims)   (tests/golden/make_golden.py)
    "1d_p2": ("1d", 2, 1, 0, 20, [8, 6, 4]),
    "1d_p3": ("1d", 3, 1, 0, 20, [8, 6, 4]),
    "15d_p4_c2": ("1.5d", 4, 2, 0, 20, [8, 6, 4]),
    "15d_p6_c2": ("1.5d", 6, 2, 0, 20, [8, 6, 4]),
    "2d_p4": ("2d", 4, 1, 0, 18, [8, 6, 4]),
    "2d_p4_b3": ("2d", 4, 1, 3, 18, [8, 6, 4]),
    "1d_p8": ("1d", 8, 1, 0, 20, [8, 6, 4]),
    "15d_p8_c2": ("1.5d", 8, 2, 0, 20, [8, 6, 4]),
    "3d_p8": ("3d", 8, 1, 0, 9, [8, 8, 4]),
}


@pytest.mark.multigpu
@pytest.mark.parametrize("kind,P,repl", [("1d", 2, 1), ("1.5d", 4, 2), ("1d", 4, 1), ("2d", 4, 1),
                                        ("3d", 8, 1)])
@pytest.mark.parametrize("dims", [[24, 8, 6], [24, 6, 8, 10]])
def test_distributed_reassociated(cg, orc, need_comm, comm, kind, P, repl, dims):
    """Narrow-first propagation on every strategy (2D/3D: row-group GEMM
    first, then SUMMA propagation of the f_out-wide U tiles); the second dims
    have widening layers (Y = Tᵀ G, G_prev = A (G Wᵀ) ⊙ relu′), one of them
    in the middle of the network."""
    need_comm(comm, P)
    model = cg.init_glorot(dims, 5, 0.5)
    out = cg.run_distributed(lambda dev: cg.generate_dataset(50, 6.0, 24, dims[-1], 2, 3, 4, device=dev),
                             model, cg.Strategy(kind, P, repl, reassociate=True), 3, comm=comm)
    od = orc.generate_dataset(50, 6.0, 24, dims[-1], 2, 3, 4)
    losses, h, y, g, w = orc.train_serial(od, dims, model.weights, 0.5, 3)
    res = dict(losses=out.losses, h_final=out.h_final, y=out.y_final, g=out.g_final,
               w=out.model.weights)
    assert max_rel_error(res, losses, h, y, g, w) < TOL


@pytest.mark.multigpu
@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("p2p,overlap,pipeline", [(True, True, False), (True, False, False),
                                                  (True, False, True), (False, False, False)])
def test_1d_exchange_paths(cg, orc, need_comm, comm, monkeypatch, P, p2p, overlap, pipeline):
    """1D stage exchanges: NVLink peer-memory pushes with the own-block SpMM
    overlapped, peer memory in one SpMM after the exchange, the pipelined form
    (per-destination pushes, per-block SpMMs as slots land; forced here by a
    zero slot threshold), and the NCCL all-gather — same numbers as the serial
    oracle over graph-replayed epochs (the flag protocol runs inside the
    replays)."""
    need_comm(comm, P)
    monkeypatch.setenv("CAGNET_PIPELINE_MIN_MB", "0" if pipeline else "1e9")
    dims = [24, 8, 8, 6]
    model = cg.init_glorot(dims, 5, 0.5)
    strat = cg.Strategy("1d", P, 1, reassociate=True, p2p=p2p, overlap=overlap)
    out = cg.run_distributed(lambda dev: cg.generate_dataset(300, 12.0, 24, 6, 2, 3, 4, device=dev),
                             model, strat, 5, comm=comm)
    od = orc.generate_dataset(300, 12.0, 24, 6, 2, 3, 4)
    losses, h, y, g, w = orc.train_serial(od, dims, model.weights, 0.5, 5)
    res = dict(losses=out.losses, h_final=out.h_final, y=out.y_final, g=out.g_final,
               w=out.model.weights)
    assert max_rel_error(res, losses, h, y, g, w) < TOL


@pytest.mark.multigpu
@pytest.mark.parametrize("P", [2, 4])
def test_1d_odd_exchange_count(cg, orc, need_comm, comm, P):
    """A widening first layer skips the last backward SpMM, leaving an odd
    number of peer-memory exchanges per epoch; the trainer evens it out with a
    flag-only exchange so the replayed epoch graph never reuses the buffer of
    the exchange before it (many replays, result still matches the oracle)."""
    need_comm(comm, P)
    dims = [8, 16, 4]
    model = cg.init_glorot(dims, 5, 0.5)
    out = cg.run_distributed(lambda dev: cg.generate_dataset(400, 12.0, 8, 4, 2, 3, 4, device=dev),
                             model, cg.Strategy("1d", P, 1, reassociate=True), 12, comm=comm)
    od = orc.generate_dataset(400, 12.0, 8, 4, 2, 3, 4)
    losses, h, y, g, w = orc.train_serial(od, dims, model.weights, 0.5, 12)
    res = dict(losses=out.losses, h_final=out.h_final, y=out.y_final, g=out.g_final,
               w=out.model.weights)
    assert max_rel_error(res, losses, h, y, g, w) < TOL


@pytest.mark.multigpu
@pytest.mark.parametrize("kind,P", [("2d", 4), ("3d", 8)])
def test_resident_sparse_tiles(cg, need_comm, comm, kind, P):
    """SUMMA with the sparse tiles kept resident after distribute(): the same
    numbers bit for bit, and no per-epoch sparse broadcast in the ledger."""
    need_comm(comm, P)
    dims = [8, 6, 4]
    model = cg.init_glorot(dims, 14, 0.5)
    outs = []
    for resident in (False, True):
        outs.append(cg.run_distributed(
            lambda dev: cg.generate_dataset(18, 4.0, dims[0], dims[-1], 11, 12, 13, device=dev),
            model, cg.Strategy(kind, P, 1, 0, resident_sparse=resident), 3, comm=comm))
    a, b = outs
    assert np.array_equal(a.losses, b.losses)
    assert np.array_equal(a.h_final, b.h_final)
    for r in range(P):
        assert b.ledger[r]["sbcast"]["calls"] == 0
        assert a.ledger[r]["sbcast"]["calls"] > 0
        for cat in ("dbcast", "reduce", "allgather"):
            assert a.ledger[r][cat] == b.ledger[r][cat]


@pytest.mark.multigpu
@pytest.mark.parametrize("name", list(DIST))
def test_distributed_matches_reference(cg, need_comm, comm, name):
    kind, P, repl, block, n, dims = DIST[name]
    need_comm(comm, P)
    gd = np.load(os.path.join(GOLD, "reference_dist.npz"))
    model = cg.init_glorot(dims, 14, 0.5)
    # The reference's own communication schedule (per-stage sparse broadcasts).
    strat = cg.Strategy(kind, P, repl, block, resident_sparse=False)
    out = cg.run_distributed(lambda dev: cg.generate_dataset(n, 4.0, dims[0], dims[-1], 11, 12, 13,
                                                             device=dev), model, strat, 3, comm=comm)
    L = len(dims)
    res = dict(losses=out.losses, h_final=out.h_final, y=out.y_final, g=out.g_final,
               w=out.model.weights)
    err = max_rel_error(res, gd[f"{name}_losses"], gd[f"{name}_h_final"],
                        [gd[f"{name}_y_{l}"] for l in range(L - 1)],
                        [gd[f"{name}_g_{l}"] for l in range(L - 1)],
                        [gd[f"{name}_w_{l}"] for l in range(L - 1)])
    assert err < TOL, err
    # Ledger reconciliation: the NCCL path meters the reference's counters exactly.
    want = gd[f"{name}_ledger"]  # [category, rank, field]
    for r in range(P):
        for ci, cat in enumerate(cg.CATEGORIES):
            got = [out.ledger[r][cat][f] for f in ("messages", "words_sent", "words_received",
                                                   "payload_words", "calls")]
            assert got == [int(x) for x in want[ci, r]], (name, r, cat)


def distributed_trainers(cg, make_data, model, strat):
    """P trainers of an in-process world on GPU 0, each created and
    distributed on its own thread (distribute() holds collectives)."""
    import threading
    P = strat.ranks
    nid = cg.comm_local_id(P, 0) if P > 1 else None
    datas = [make_data() for _ in range(P)]
    trainers, errors = [None] * P, []

    def body(r):
        try:
            t = cg.Trainer(datas[r], model, strat, r, nid)
            t.distribute()
            trainers[r] = t
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)
            cg.comm_local_abort(nid, str(e))

    th = [threading.Thread(target=body, args=(r,)) for r in range(P)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errors, errors
    return trainers, datas


@pytest.mark.parametrize("kind,P,repl", [("1d", 8, 1), ("1.5d", 8, 2), ("2d", 4, 1), ("3d", 8, 1)])
def test_trainer_parts_match_reference_distribute(cg, ref, kind, P, repl):
    """Trainer::distribute() of the product (every rank's own a_parts /
    at_parts, read back through cagnet_trainer_part) against the reference's
    distribute() (dist_1d.cpp:28-44, dist_15d.cpp:32-47, dist_2d.cpp:41-54,
    dist_3d.cpp:39-55) on config 1: structure bit-exact, values (float) of
    the reference's doubles, per-part nnz equal to the committed golden."""
    gold = np.load(os.path.join(GOLD, "reference_config1.npz"))[f"parts_{kind}_p{P}"]
    dims = [128, 16, 8]
    model = cg.init_glorot(dims, 4, 0.5)
    strat = cg.Strategy(kind, P, repl)
    trainers, _ = distributed_trainers(
        cg, lambda: cg.generate_dataset(4096, 16.0, 128, 8, 1, 2, 3, device=0), model, strat)
    rdata = ref.dataset(4096, 16.0, 128, 8, 1, 2, 3)
    rt = ref.distribute(rdata, ref.model(dims, 4, 0.5), kind, P, repl)
    rows = []
    for r, t in enumerate(trainers):
        assert t.num_parts() == rt.num_parts(r)
        for q in range(t.num_parts()):
            nnz = []
            for which in (0, 1):
                rp, ci, v = t.part(which, q).download()
                want = rt.part(r, which, q)
                assert np.array_equal(rp, want.row_ptr), (kind, r, q, which)
                assert np.array_equal(ci, want.col_idx), (kind, r, q, which)
                assert np.array_equal(v, want.vals.astype(np.float32)), (kind, r, q, which)
                nnz.append(len(ci))
            rows.append([r, q] + nnz)
    assert np.array_equal(np.asarray(rows), gold)


@pytest.mark.parametrize("panel_mb,passes", [(0.4, 2), (0.15, 5), (0.06, 12)])
def test_l2_multipass_spmm_matches_serial(cg, orc, monkeypatch, panel_mb, passes):
    """L2 column-blocked SpMM (trainer.cu spmm_passes: one pass per column
    block when the gathered panel exceeds the L2 budget and rows carry >= 64
    nonzeros): forced to 2 / 5 / 12 passes by shrinking the budget; the
    reference propagation order keeps the f = 64 SpMM, which blocks."""
    n, deg, dims = 3000, 150.0, [64, 16, 8]
    model = cg.init_glorot(dims, 5, 0.5)
    od = orc.generate_dataset(n, deg, dims[0], dims[-1], 2, 3, 4)
    losses, h, y, g, w = orc.train_serial(od, dims, model.weights, 0.5, 2)
    launches = {}
    for mb in (1e6, panel_mb):
        monkeypatch.setenv("CAGNET_L2_PANEL_MB", str(mb))
        data = cg.generate_dataset(n, deg, dims[0], dims[-1], 2, 3, 4)
        t = cg.make_trainer(data, model, cg.Strategy("1d", 1, graph=False))
        t.distribute()
        got = list(t.run_epochs(1))  # first epoch also builds the column blocks
        k0 = cg.kernel_launches()
        got += list(t.run_epochs(1))
        launches[mb] = cg.kernel_launches() - k0
        L = len(dims)
        out = dict(losses=got, h_final=t.h_tile(L - 1).astype(np.float64),
                   y=[t.y(l).astype(np.float64) for l in range(L - 1)],
                   g=[t.g_tile(l).astype(np.float64) for l in range(L - 1)],
                   w=[t.weight(l).astype(np.float64) for l in range(L - 1)])
        assert max_rel_error(out, losses, h, y, g, w) < TOL, mb
    # Passes per SpMM (trainer.cu spmm_passes): ceil(panel / budget), at most
    # 64 and at most nnz-per-row / 12.  Per epoch the reference order runs
    # SpMMs of width 64 and 16 forward and 8 and 16 backward.
    def nb(f):
        import math
        per_row = (od["adj"].nnz) / n
        return max(1, min(64, math.ceil(n * f * 4 / (panel_mb * 1048576)), int(per_row / 12)))
    assert nb(64) == passes
    extra = sum(nb(f) - 1 for f in (64, 16, 8, 16))
    assert launches[panel_mb] - launches[1e6] == extra, launches


def on_all_ranks(trainers, fn):
    """fn(trainer) on every rank concurrently (collective calls)."""
    import threading
    errors = []

    def body(t):
        try:
            fn(t)
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    th = [threading.Thread(target=body, args=(t,)) for t in trainers]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errors, errors


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("layers", [[1], [1, 2], [2, 1, 2]])
def test_forward_layer_between_replayed_epochs(cg, orc, P, layers):
    """run_forward_layer (dist_common.cpp:110-115) between CUDA-graph epochs on
    the 1D peer-memory exchange: the layer's direct push is settled and the
    buffer rotation padded, so the replays that follow still match the
    serial oracle (forward_layer recomputes activations from the same
    weights, so it leaves the training trajectory unchanged)."""
    dims = [24, 8, 8, 6]
    model = cg.init_glorot(dims, 5, 0.5)
    strat = cg.Strategy("1d", P, 1, reassociate=True)
    trainers, _ = distributed_trainers(
        cg, lambda: cg.generate_dataset(300, 12.0, 24, 6, 2, 3, 4, device=0), model, strat)
    losses = {t.rank: [] for t in trainers}
    on_all_ranks(trainers, lambda t: losses[t.rank].extend(t.run_epochs(3)))
    for l in layers:
        on_all_ranks(trainers, lambda t: t.forward_layer(l))
    on_all_ranks(trainers, lambda t: losses[t.rank].extend(t.run_epochs(4)))
    od = orc.generate_dataset(300, 12.0, 24, 6, 2, 3, 4)
    ref_losses, h, y, g, w = orc.train_serial(od, dims, model.weights, 0.5, 7)
    L = len(dims)
    for t in trainers:
        r0, r1 = t.tile_rows(t.rank)
        assert np.allclose(losses[t.rank], ref_losses, rtol=TOL, atol=TOL)
        import oracle
        assert oracle.rel_frobenius(t.weight(0), w[0]) < TOL
        assert oracle.rel_frobenius(t.h_tile(L - 1), h[r0:r1]) < TOL


@pytest.mark.parametrize("graph", [True, False])
def test_host_steps_sync_and_pipelined(cg, graph):
    """The end-to-end call (cagnet_trainer_step_host: H2D of the rank's inputs,
    the epoch, D2H of the loss) and its pipelined form (prefetch_host +
    step_prefetched, step k+1's copies overlapping step k's epoch) give the same
    losses bit for bit, alternating two different input sets; the first step
    on the dataset's own inputs equals run_epochs."""
    dims = [24, 8, 6]
    data = cg.generate_dataset(300, 12.0, 24, 6, 2, 3, 4)
    model = cg.init_glorot(dims, 5, 0.5)
    strat = cg.Strategy("1d", 1, reassociate=True, graph=graph)
    x1 = np.ascontiguousarray(data.features(), np.float32)
    l1 = np.ascontiguousarray(data.labels(), np.int32)
    x2 = np.ascontiguousarray(x1 * 0.5 + 0.25, np.float32)
    l2 = np.ascontiguousarray((l1 + 1) % 6, np.int32)
    seq = [(x1, l1), (x2, l2), (x1, l1), (x2, l2), (x2, l2)]

    def fresh():
        t = cg.make_trainer(data, model, strat)
        t.distribute()
        return t

    ref = fresh().run_epochs(1)[0]
    a = fresh()
    sync = [a.step_host(x, l) for x, l in seq]
    b = fresh()
    piped = []
    b.prefetch_host(*seq[0])
    for k in range(len(seq)):
        if k + 1 < len(seq):
            b.prefetch_host(*seq[k + 1])
        piped.append(b.step_prefetched())
    assert sync[0] == ref
    assert sync == piped
    assert len(set(sync)) > 1
    with pytest.raises(cg.CagnetError, match="no staged inputs"):
        b.step_prefetched()
