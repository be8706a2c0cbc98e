"""Parity helpers: run a workload through the lmfao_gpu C-ABI and compare with
the oracle (keys/counts bit-exact; floats per DESIGN.md reading R14)."""
import numpy as np

import oracle
import synth
from _udaf import float_close


def run_gpu(db, batch, shard=None, engine_kw=None, runs=1, info=False, cols=None):
    """cols: optional relation -> columns override (e.g. pinned torch tensors: deferred load)."""
    from paper_1906_08687_b200 import lmfao
    e = lmfao.Engine(**(engine_kw or {}))
    try:
        for r in db.relations:
            e.add_relation(r.name, cols[r.name] if cols else r.cols)
        e.set_join_tree(db.root, db.edges)
        if shard is not None:
            e.set_root_shard(*shard)
        e.prepare()
        qids = [e.add_query(q.groupby, q.udafs) for q in batch]
        e.plan()
        for _ in range(runs):
            e.run()
        out = [e.fetch(q) for q in qids]
        if info:
            return out, e.plan_info()
        return out
    finally:
        e.close()


def integral_udaf(u):
    """UDAF whose every product has an integral coefficient and only constant-integer or
    predicate factors: its sum is an integer and must match exactly."""
    for p in u:
        if float(p.coeff) != int(p.coeff):
            return False
        for f in p.factors:
            if f.kind == synth.F_IDENT:
                return False
            if f.kind == synth.F_CONST and float(f.param) != int(f.param):
                return False
    return True


def assert_parity(gpu, ref, batch, rel=1e-9):
    for qi, ((k, v, c), r, q) in enumerate(zip(gpu, ref, batch)):
        assert k.shape == r.keys.shape, (qi, k.shape, r.keys.shape)
        assert np.array_equal(k.astype(np.int64), r.keys), f"query {qi}: group keys differ"
        assert np.array_equal(c, r.counts), f"query {qi}: counts differ"
        assert v.shape == r.vals.shape
        for j, u in enumerate(q.udafs):
            if integral_udaf(u):
                assert np.array_equal(v[:, j], r.vals[:, j]), f"query {qi} udaf {j}: integral sums differ"
        ok = float_close(v, r.vals, r.absmass, rel=rel)
        if not ok.all():
            bad = np.argwhere(~ok)[:5]
            raise AssertionError(f"query {qi}: {int((~ok).sum())} values out of tolerance, e.g. "
                                 + "; ".join(f"[{a},{b}] gpu={v[a, b]!r} oracle={r.vals[a, b]!r}" for a, b in bad))
