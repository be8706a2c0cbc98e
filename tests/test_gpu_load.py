"""Loading through LMFAO_COLS_HOST_DEFERRED (include/lmfao_gpu.h lmfao_add_relation): pinned
host columns streamed in by lmfao_prepare on a copy stream, overlapped with the remap, sort
and permutation.  Results must equal the synchronous-copy load (keys and counts bit for bit) and match the
oracle, on multi-level trees, with dangling keys (row compaction), and with root sharding."""
import numpy as np
import pytest
import torch

import oracle
import synth
from _parity import assert_parity, run_gpu

pytestmark = pytest.mark.gpu


def pinned(db):
    return {r.name: {c: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for c, v in r.cols.items()}
            for r in db.relations}


def same(a, b):
    """Keys and counts bit-exact; sums up to summation order (the covariance scan assigns
    work items to warps dynamically, so its fp64 partial sums are not bit-reproducible)."""
    for (k1, v1, c1), (k2, v2, c2) in zip(a, b):
        assert np.array_equal(k1, k2) and np.array_equal(c1, c2)
        assert np.allclose(v1, v2, rtol=1e-12, atol=1e-12)


CASES = {
    "c1": lambda: (synth.config1().db, synth.config1().batch),
    "c2_small": lambda: (lambda w: (w.db, w.batch))(synth.config2(fact_rows=50_000, dim_rows=(50, 500, 5_000))),
    "c3_small": lambda: (lambda w: (w.db, w.batch))(synth.config3(fact_rows=40_000, dim_rows=(40, 300, 2_000))),
    "h2_dangling": lambda: (synth.hand_h2(), synth.random_batch(7, synth.hand_h2())),
    "random_tree": lambda: (lambda db: (db, synth.random_batch(3, db, groupby_ok=lambda a: a in db.rel(db.root).cols)))(
        synth.random_db(11, max_rels=5, max_rows=3000)),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_deferred_load_equals_sync_load(case):
    db, batch = CASES[case]()
    sync = run_gpu(db, batch)
    deferred = run_gpu(db, batch, cols=pinned(db))
    same(sync, deferred)
    assert_parity(deferred, oracle.evaluate(db, batch), batch)


def test_deferred_load_sharded():
    w = synth.config2(fact_rows=30_011, dim_rows=(30, 300, 3_000))
    cols = pinned(w.db)
    for p in range(3):
        same(run_gpu(w.db, w.batch, shard=(p, 3)), run_gpu(w.db, w.batch, shard=(p, 3), cols=cols))


def test_bad_load_mode_rejected():
    from paper_1906_08687_b200 import lmfao
    e = lmfao.Engine()
    try:
        import ctypes
        names = (ctypes.c_char_p * 1)(b"a")
        dt = (ctypes.c_int32 * 1)(lmfao.INT32)
        buf = np.zeros(4, np.int32)
        cp = (ctypes.c_void_p * 1)(buf.ctypes.data)
        rid = ctypes.c_int32()
        s = lmfao._lib.lmfao_add_relation(e.h, b"R", 4, 1, names, dt, cp, 3, ctypes.byref(rid))
        assert lmfao.STATUS[s] == "LMFAO_ERR_INVALID_ARG"
    finally:
        e.close()


@pytest.mark.parametrize("seed", [0, 2, 4, 6])
def test_deferred_load_multi_root(seed):
    """Deferred columns may still be in flight when prepare returns (plan waits for them); a
    query placed at another root copies every relation into a secondary context inside
    add_query, which must wait for the copies first.  Pinned (deferred) columns vs the oracle,
    on random trees whose batches use other roots."""
    from paper_1906_08687_b200 import lmfao
    db = synth.random_db(300 + seed, max_rels=5, max_rows=60_000, unique_child_keys=True)
    ints = {a for r in db.relations for a, v in r.cols.items() if v.dtype == np.int32}
    batch = synth.random_batch(seed, db, n_queries=5, groupby_ok=lambda a: a in ints)
    ref = oracle.evaluate(db, batch)
    cols = pinned(db)
    e = lmfao.Engine()
    try:
        for r in db.relations:
            e.add_relation(r.name, cols[r.name])
        e.set_join_tree(db.root, db.edges)
        e.prepare()
        kept = []
        for qi, q in enumerate(batch):
            try:
                kept.append((qi, e.add_query(q.groupby, q.udafs)))
            except lmfao.LmfaoError as ex:
                assert ex.name == "LMFAO_ERR_UNSUPPORTED", ex
        e.plan()
        e.run()
        got = [e.fetch(q) for _, q in kept]
    finally:
        e.close()
    assert kept
    assert_parity(got, [ref[qi] for qi, _ in kept], [batch[qi] for qi, _ in kept])
