"""The exported collective seams (cagnet_comm_*, RankContext runtime.hpp:55-96)
against the reference's SimRuntime running the same script
(oracle/ref_shim.cpp ref_collectives_script): results and the ledger counters
of every rank, category by category.  The ranks are threads of this process on
one GPU (in-process world); with enough GPUs the NCCL variant runs too."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [("2d", 4, 1), ("1.5d", 4, 2), ("3d", 8, 1), ("1.5d", 6, 2)]


@pytest.mark.parametrize("kind,P,repl", CASES)
def test_collective_seams_match_reference(cg, ref, need_comm, comm, kind, P, repl):
    need_comm(comm, P)
    import torch
    want_led, want_rs, want_ag = ref.collectives_script(kind, P, repl)
    nid = cg.comm_local_id(P, 0) if comm == "local" else cg.comm_unique_id()
    strat = cg.Strategy(kind, P, repl)
    results, errors = {}, []

    def body(r):
        try:
            dev = 0 if comm == "local" else r
            torch.cuda.set_device(dev)
            c = cg.Comm(strat, r, nid, dev)
            st = torch.cuda.Stream(device=dev)
            s = st.cuda_stream
            row, col = c.group("row"), c.group("col")
            with torch.cuda.stream(st):
                m = (r + 1 + 0.01 * torch.arange(15, dtype=torch.float32, device=dev)).reshape(3, 5)
                b = m.clone() if r == row[0] else torch.zeros(3, 5, device=dev)
                c.bcast("row", row[0], b.data_ptr(), 15, "f32", "dbcast", s)
                x = (r + 0.5 * torch.arange(8, dtype=torch.float32, device=dev)).reshape(2, 4)
                c.all_reduce("world", x.data_ptr(), 8, "f32", "reduce", s)
                sc = torch.tensor([r * 1.5], dtype=torch.float64, device=dev)
                c.all_reduce("world", sc.data_ptr(), 1, "f64", "reduce", s)
                counts = [3] + [1] * (len(col) - 1)
                y = (r * 0.25 + torch.arange(3 * sum(counts), dtype=torch.float32, device=dev))
                rs = torch.zeros(counts[col.index(r)] * 3, device=dev)
                c.reduce_scatter_rows("col", y.data_ptr(), rs.data_ptr(), counts, 3, "reduce", s)
                rc = [2] + [1] * (len(row) - 1)
                z = 100.0 * r + torch.arange(3 * rc[row.index(r)], dtype=torch.float32, device=dev)
                ag = torch.zeros(3 * sum(rc), device=dev)
                c.all_gather_rows("row", z.data_ptr(), ag.data_ptr(), rc, 3, "allgather", s)
                rp = torch.tensor([0, 2, 2, 4], dtype=torch.int64, device=dev)
                ci = torch.tensor([0, 3, 1, 2], dtype=torch.int32, device=dev)
                va = torch.tensor([1.0, 2.0, 3.0, 4.0], device=dev)
                if r != row[-1]:
                    rp.zero_(), ci.zero_(), va.zero_()
                c.bcast_csr("row", row[-1], rp.data_ptr(), 3, ci.data_ptr(), va.data_ptr(), 4, "sbcast", s)
                if kind == "3d":
                    f = torch.full((3,), float(r), device=dev)
                    c.all_reduce("fiber", f.data_ptr(), 3, "f32", "reduce", s)
            st.synchronize()
            results[r] = dict(b=b.cpu().numpy(), x=x.cpu().numpy(), sc=float(sc.item()),
                              rs=rs.cpu().numpy(), ag=ag.cpu().numpy(), rp=rp.cpu().numpy(),
                              ci=ci.cpu().numpy(), va=va.cpu().numpy(), ledger=c.ledger(),
                              row=row)
            c.free()
        except Exception as e:  # pragma: no cover - reported below
            errors.append((r, e))
            if comm == "local":
                cg.comm_local_abort(nid, str(e))

    th = [threading.Thread(target=body, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    xsum = sum((q + 0.5 * np.arange(8)) for q in range(P)).reshape(2, 4)
    for r in range(P):
        res = results[r]
        root = res["row"][0]
        assert np.allclose(res["b"], (root + 1 + 0.01 * np.arange(15)).reshape(3, 5))
        assert np.allclose(res["x"], xsum)
        assert res["sc"] == sum(q * 1.5 for q in range(P))
        assert np.allclose(res["rs"], want_rs[r][:res["rs"].size], rtol=1e-6)
        assert np.allclose(res["ag"], want_ag[r][:res["ag"].size], rtol=1e-6)
        assert list(res["rp"]) == [0, 2, 2, 4] and list(res["ci"]) == [0, 3, 1, 2]
        assert list(res["va"]) == [1.0, 2.0, 3.0, 4.0]
        for ci_, cat in enumerate(cg.CATEGORIES):
            got = [res["ledger"][cat][f] for f in ("messages", "words_sent", "words_received",
                                                 "payload_words", "calls")]
            assert got == [int(v) for v in want_led[ci_, r]], (kind, r, cat)
