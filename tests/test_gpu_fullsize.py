"""Parity at BASELINE.json's full sizes, in the configuration bench.py times: the
whole batch runs on the GPU, and a seeded sample of its outputs is recomputed by
the oracle one query at a time (plus properties that hold at any size)."""
import numpy as np
import pytest

import oracle
import synth
from _parity import assert_parity, run_gpu
from _udaf import float_close

pytestmark = pytest.mark.gpu


def _sample(batch, qi, n, seed):
    rng = np.random.default_rng(seed)
    q = batch[qi]
    idx = sorted(rng.choice(len(q.udafs), size=min(n, len(q.udafs)), replace=False).tolist())
    return idx, synth.Query(list(q.groupby), [q.udafs[i] for i in idx])


def _check_sampled(w, qi, n, seed=0):
    gpu = run_gpu(w.db, w.batch)
    idx, q = _sample(w.batch, qi, n, seed)
    ref = oracle.evaluate(w.db, [q])[0]
    k, v, c = gpu[qi]
    assert np.array_equal(k.astype(np.int64), ref.keys)
    assert np.array_equal(c, ref.counts)
    ok = float_close(v[:, idx], ref.vals, ref.absmass)
    assert ok.all(), (np.argwhere(~ok)[:5], v[:, idx][~ok][:5], ref.vals[~ok][:5])
    return gpu


def test_c2_full_all_780_outputs():
    """BASELINE.json configs[1] at its full size, in the launch configuration bench.py times:
    every one of the 780 aggregates against the oracle over the whole 10M-row join
    (OpenMP chunks on the host cores; SURVEY.md §8(c) "GPU acceptance")."""
    w = synth.config2()
    gpu = run_gpu(w.db, w.batch)
    ref = oracle.evaluate(w.db, w.batch, threads=0)
    assert_parity(gpu, ref, w.batch)
    assert int(gpu[0][2][0]) == 10_000_000


def test_c3_full_sampled_outputs():
    w = synth.config3()
    gpu = _check_sampled(w, len(w.batch) - 1, 30)
    # categorical queries: counts per category sum to the fact rows; one checked fully
    ref = oracle.evaluate(w.db, [w.batch[0]])[0]
    k, v, c = gpu[0]
    assert np.array_equal(k.astype(np.int64), ref.keys) and np.array_equal(c, ref.counts)
    assert float_close(v, ref.vals, ref.absmass).all()
    for qi in range(len(w.batch) - 1):
        assert int(gpu[qi][2].sum()) == 10_000_000


def test_c4_full_sampled_queries():
    w = synth.config4()
    gpu = run_gpu(w.db, w.batch)
    rng = np.random.default_rng(1)
    for qi in sorted(rng.choice(len(w.batch), size=5, replace=False).tolist()) + [len(w.batch) - 1]:
        ref = oracle.evaluate(w.db, [w.batch[qi]])[0]
        k, v, c = gpu[qi]
        assert np.array_equal(k.astype(np.int64), ref.keys), qi
        assert np.array_equal(c, ref.counts), qi
        assert np.array_equal(v[:, 0], ref.vals[:, 0]), qi
    # marginals of every pair table equal the single-attribute counts (any size)
    names = w.meta["attrs"]
    single = {q.groupby[0]: gpu[i] for i, q in enumerate(w.batch) if len(q.groupby) == 1}
    for i, q in enumerate(w.batch):
        if len(q.groupby) != 2:
            continue
        k, v, c = gpu[i]
        for pos in (0, 1):
            sk, sv, sc = single[q.groupby[pos]]
            vals, inv = np.unique(k[:, pos], return_inverse=True)
            tot = np.bincount(inv, weights=c.astype(np.float64))
            assert np.array_equal(vals, sk[:, 0]) and np.array_equal(tot.astype(np.uint64), sc)
