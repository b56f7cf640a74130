"""Failure detection (the reference's deadlock detector raises
SimError instead of hanging, runtime.cpp:58-136): a failed or silent rank
surfaces as an exception on its peers, never as a hung GPU or a trapped
context."""
import threading
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_rank_failure_releases_peers(cg, need_gpus):
    """Rank 1 raises before joining; ranks 0, 2, 3, already blocked in
    distribute()'s collectives, are released by its abort with the reason."""
    need_gpus(1)
    nid = cg.comm_local_id(4, 0)
    model = cg.init_glorot([8, 6, 4], 5, 0.5)
    strat = cg.Strategy("2d", 4, 1)
    errors = {}

    def body(r):
        try:
            if r == 1:
                raise ValueError("dataset for rank 1 failed")
            d = cg.generate_dataset(40, 6.0, 8, 4, 1, 2, 3, device=0)
            t = cg.Trainer(d, model, strat, r, nid)
            t.distribute()
        except Exception as e:
            errors[r] = e
            if r == 1:
                cg.comm_local_abort(nid, f"rank {r} raised: {e}")

    t0 = time.time()
    th = [threading.Thread(target=body, args=(r,)) for r in range(4)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert time.time() - t0 < 60
    assert isinstance(errors[1], ValueError)
    for r in (0, 2, 3):
        assert "aborted" in str(errors[r]) and "rank 1 raised" in str(errors[r]), errors[r]


def test_run_distributed_invalid_model_raises(cg, need_gpus):
    """A model that does not fit the dataset fails on every rank at
    construction; run_distributed raises the reference's error, no hang."""
    need_gpus(1)
    d = cg.generate_dataset(40, 6.0, 8, 4, 1, 2, 3, device=0)
    model = cg.init_glorot([9, 6, 4], 5, 0.5)
    with pytest.raises(cg.InvalidArgument, match="input width 9"):
        cg.run_distributed(d, model, cg.Strategy("3d", 8), 1, comm="local")


def test_silent_rank_times_out_without_trap(cg, need_gpus, monkeypatch):
    """Both ranks capture their epoch graph; then only rank 0 keeps replaying.
    Its device-side waits for rank 1's flags time out (budget lowered to
    300 ms), record the failure in the host-mapped error word and return;
    the host raises CAGNET_ENCCL and the CUDA context stays usable."""
    need_gpus(1)
    monkeypatch.setenv("CAGNET_WAIT_TIMEOUT_MS", "300")
    nid = cg.comm_local_id(2, 0)
    datas = [cg.generate_dataset(60, 6.0, 8, 4, 1, 2, 3, device=0) for _ in range(2)]
    model = cg.init_glorot([8, 6, 4], 5, 0.5)
    strat = cg.Strategy("1d", 2, 1, reassociate=True)
    trainers, errors = [None, None], []

    def body(r):
        try:
            t = cg.Trainer(datas[r], model, strat, r, nid)
            t.distribute()
            t.run_epochs(3)  # eager, captured, replayed
            trainers[r] = t
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    th = [threading.Thread(target=body, args=(r,)) for r in range(2)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errors, errors
    with pytest.raises(cg.CagnetError) as ei:
        trainers[0].run_epochs(1)
    assert ei.value.code == 3 and "timed out" in str(ei.value), str(ei.value)
    # The context survived: a fresh single-rank run still trains.
    d = cg.generate_dataset(32, 8.0, 16, 4, 1, 2, 3, device=0)
    t = cg.make_trainer(d, cg.init_glorot([16, 16, 4], 4, 0.5), cg.Strategy("1d", 1))
    t.distribute()
    losses = t.run_epochs(2)
    assert np.all(np.isfinite(losses))
