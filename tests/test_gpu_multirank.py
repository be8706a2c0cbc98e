"""The multi-GPU path of lmfao_gpu on one GPU: `world` contexts of one process form an
in-process loopback group (lmfao_create_loopback), one host thread per rank.  Every rank
passes the whole root, keeps its shard of the sorted root (lmfao_prepare), and runs the same
kernels as an NCCL rank — all-reduce of small outputs, reduce-scatter of large dense tables,
the peer-memory exchange of sparse cuboids — with host barriers between the phases of a run
(no kernel waits for another rank's kernel).  Checked against the oracle over the whole root:
  * replicated outputs are complete and equal on every rank;
  * a distributed output holds, on each rank, exactly the oracle's groups whose cell lies in
    the rank's lmfao_owner_range; lmfao_gather_result assembles the full table, in canonical
    order, on the chosen root rank;
  * repeated runs (the exchange's run-parity buffers and epoch flags) give the same results."""
import threading

import numpy as np
import pytest

import oracle
import synth
from _parity import assert_parity
from _udaf import float_close

pytestmark = pytest.mark.gpu

_GROUP = [0]


def _run_ranks(db, batch, world, runs=2, gather_root=None):
    from paper_1906_08687_b200 import lmfao
    _GROUP[0] += 1
    name = f"t{_GROUP[0]}"
    out = [None] * world
    errs = []
    bar = threading.Barrier(world)

    def rank_main(r):
        try:
            e = lmfao.Engine(rank=r, world=world, loopback=name)
            try:
                qids = lmfao.load(e, db, batch)
                e.plan()
                res = []
                for _ in range(runs):
                    e.run()
                    res.append([e.fetch(q) for q in qids])
                info = e.plan_info()
                gathered = None
                if gather_root is not None:
                    for q in qids:
                        e.gather_result(q, gather_root)
                    gathered = [e.fetch(q) for q in qids]
                bar.wait()
                out[r] = (res, info, gathered)
            finally:
                e.close()
        except Exception as ex:  # pragma: no cover
            errs.append((r, repr(ex)))
            bar.abort()

    ts = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(600)
    assert not errs, errs
    return out


def _cells(keys, q, db):
    """Cell index of each group key (mixed radix over the sorted distinct values of each
    group-by attribute in the whole database, the engine's dictionaries)."""
    cell = np.zeros(len(keys), dtype=np.int64)
    for i, a in enumerate(q.groupby):
        dom = np.unique(np.concatenate([r.cols[a] for r in db.relations if a in r.cols and r.name == _owner(db, a)]))
        cell = cell * len(dom) + np.searchsorted(dom, keys[:, i])
    return cell


def _owner(db, a):
    for r in db.relations:  # the root first, then the children (top-most holder)
        if a in r.cols:
            return r.name


def _ncells(q, db):
    n = 1
    for a in q.groupby:
        n *= len(np.unique(db.rel(_owner(db, a)).cols[a]))
    return n


def _check_ranks(db, batch, out, world, gather_root):
    from paper_1906_08687_b200 import lmfao
    ref = oracle.evaluate(db, batch, threads=0)
    placements = set()
    for r in range(world):
        res, info, gathered = out[r]
        assert info["world"] == world and info["rank"] == r and info["comm"] == "loopback"
        for run in res:
            for qi, (q, rr, (k, v, c)) in enumerate(zip(batch, ref, run)):
                pl = info["outputs"][qi]["placement"]
                placements.add(pl)
                if pl == "replicated":
                    assert_parity([(k, v, c)], [rr], [q])
                    continue
                lo, hi = lmfao.owner_range(_ncells(q, db), r, world)
                assert info["outputs"][qi]["cells"] == [lo, hi]
                cells = _cells(rr.keys, q, db)
                sel = (cells >= lo) & (cells < hi)
                assert np.array_equal(k.astype(np.int64), rr.keys[sel]), (qi, r)
                assert np.array_equal(c, rr.counts[sel]), (qi, r)
                assert float_close(v, rr.vals[sel], rr.absmass[sel]).all(), (qi, r)
        if r == gather_root:
            assert_parity(gathered, ref, batch)
        # a re-run reproduces the same bits (fixed-order sums, deterministic exchange merge order)
        for a, b in zip(res[0], res[-1]):
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[2], b[2])
    return placements


@pytest.mark.parametrize("world", [2, 3])
def test_multirank_covariance_allreduce(world):
    w = synth.config2(fact_rows=30_011, dim_rows=(30, 200, 1500))
    out = _run_ranks(w.db, w.batch, world, runs=3, gather_root=0)
    assert _check_ranks(w.db, w.batch, out, world, 0) == {"replicated"}
    # every rank holds the same bits
    for r in range(1, world):
        assert np.array_equal(out[r][0][-1][0][1], out[0][0][-1][0][1])


@pytest.mark.parametrize("world", [2, 4])
def test_multirank_counts_reduce_scatter(world, monkeypatch):
    """C4-shaped pairwise counts; tables of >= 64 cells reduce-scattered by cell range."""
    monkeypatch.setenv("LMFAO_DIST_CELLS", "64")
    w = synth.config4(fact_rows=20_011, dim_rows=(20, 60, 200))
    batch = [q for q in w.batch if len(q.groupby) == 2][:12] + [q for q in w.batch if len(q.groupby) < 2][:4]
    out = _run_ranks(w.db, batch, world, runs=2, gather_root=world - 1)
    pl = _check_ranks(w.db, batch, out, world, world - 1)
    assert "reduce_scattered" in pl and "replicated" in pl


@pytest.mark.parametrize("world", [2, 3])
def test_multirank_cube_sparse_exchange(world, monkeypatch):
    """C5-shaped cube + covariance: the {A,B,C} cuboid (and {B,C}) exchanged through peer memory
    as sparse records, cuboids rolled up from it and the large dense ones reduce-scattered,
    small ones and the covariance all-reduced."""
    monkeypatch.setenv("LMFAO_CUBE_SPARSE_CELLS", "2000")
    monkeypatch.setenv("LMFAO_DIST_CELLS", "200")
    w = synth.config5(fact_rows=40_011, dim_rows=(40, 300, 2000, 9000), cube_doms=(7, 30, 100))
    out = _run_ranks(w.db, w.batch, world, runs=3, gather_root=0)
    pl = _check_ranks(w.db, w.batch, out, world, 0)
    assert {"exchanged", "reduce_scattered", "replicated"} <= pl, pl
