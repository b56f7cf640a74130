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
    """Rank 1 raises before its first collective; rank 0, already waiting in
    the rendezvous, is released and the original error is reported."""
    need_gpus(1)

    def factory(dev, calls=[0]):
        calls[0] += 1
        if calls[0] == 2:
            raise ValueError("dataset for rank 1 failed")
        return cg.generate_dataset(40, 6.0, 8, 4, 1, 2, 3, device=dev)

    model = cg.init_glorot([8, 6, 4], 5, 0.5)
    t0 = time.time()
    with pytest.raises(ValueError, match="rank 1 failed"):
        cg.run_distributed(factory, model, cg.Strategy("2d", 4, 1), 2, comm="local")
    assert time.time() - t0 < 60


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
