"""Parity of the histogram path for regression-tree node batches (rt.cu, §8 row (e)):
threshold-cell histograms of w = (1, y, y^2) over the root, fact->dimension views, and
dimension-side finishing, against the oracle.  Covers every Kronecker operator on root
and dimension attributes (fp64 and int32), thresholds that coincide with data values
(the exact-equality cells), group-bys on root and dimension attributes, batches without
a target attribute, coefficients and sums of products, ragged and tiny row counts."""
import numpy as np
import pytest

import oracle
import synth
from _parity import assert_parity, run_gpu
from synth import F_EQ, F_GE, F_GT, F_LE, F_LT, F_NE, Factor, Product, Query, ident

pytestmark = pytest.mark.gpu

OPS = [F_LT, F_LE, F_GT, F_GE, F_EQ, F_NE]


def rt_db(seed, n, dim_rows=(30, 200, 1500), s=1.1, dyadic=True):
    """C3-shaped snowflake: fact F(k1..k3, x1, x2 fp64, i1 int32, c1 int32, y fp64), dims
    D_r(k_r, d_r fp64, e_r int32, g_r int32 categorical)."""
    rng = np.random.default_rng(seed)
    F = {}
    dims = []
    for r, nr in enumerate(dim_rows, start=1):
        keys = synth.distinct_keys(synth._rng(seed, "RT", r), nr)
        d = rng.standard_normal(nr)
        if dyadic:
            d = np.round(d * 4) / 4  # values on the threshold grid -> equality cells are hit
        dims.append(synth.Relation(f"D{r}", {f"k{r}": keys, f"d{r}": d,
                                              f"e{r}": rng.integers(-3, 4, nr).astype(np.int32),
                                              f"g{r}": rng.integers(0, 5 + 7 * r, nr).astype(np.int32)}))
        F[f"k{r}"] = synth.zipf_fk(seed, "F", f"k{r}", keys, s, n)
    x1 = rng.standard_normal(n)
    F["x1"] = np.round(x1 * 8) / 8 if dyadic else x1
    F["x2"] = rng.standard_normal(n)
    F["i1"] = rng.integers(-5, 6, n).astype(np.int32)
    F["c1"] = rng.integers(0, 9, n).astype(np.int32)
    F["c2"] = rng.integers(0, 600, n).astype(np.int32)
    F["y"] = rng.standard_normal(n)
    db = synth.Database([synth.Relation("F", F)] + dims, "F", [("F", d.name) for d in dims])
    return db


def c3_like(db, thresholds, attrs, cats):
    return synth.rt_batch(attrs, "y", cats, thresholds)


@pytest.mark.parametrize("n", [1, 7, 31, 32, 33, 1000, 30_011])
def test_rt_c3_shape_ragged(n):
    db = rt_db(1, n)
    batch = c3_like(db, synth.thresholds_c3(), ["x1", "x2", "d1", "d2", "d3"], ["c1", "c2", "g1", "g2", "g3"])
    gpu, info = run_gpu(db, batch, info=True)
    assert info["fast_path"] and info["fast_path"]["kind"] == "rt", info
    assert_parity(gpu, oracle.evaluate(db, batch), batch)


def test_rt_every_operator_root_and_dim_int_and_float():
    db = rt_db(2, 20_000)
    udafs = [[Product(1.0, ())], [Product(1.0, (ident("y"),))]]
    for a, ts in [("x1", [-1.0, 0.0, 0.125, 2.5]), ("i1", [-2, 0, 3]), ("d2", [-0.5, 0.0, 0.25]),
                  ("e3", [-1, 0, 2]), ("x2", [0.0])]:
        for op in OPS:
            for t in ts:
                p = Factor(op, a, float(t))
                udafs.append([Product(1.0, (p,))])
                udafs.append([Product(2.0, (ident("y"), p)), Product(-1.0, (ident("y"), ident("y"), p))])
    batch = [Query([], udafs)]
    gpu, info = run_gpu(db, batch, info=True)
    assert info["fast_path"]["kind"] == "rt"
    assert_parity(gpu, oracle.evaluate(db, batch), batch)


def test_rt_groupbys_without_target_and_with_coefficients():
    db = rt_db(3, 25_000)
    batch = [Query(["c2"], [[Product(1.0, ())], [Product(3.0, ())], [Product(0.5, (ident("y"), ident("y")))]]),
             Query(["g3"], [[Product(1.0, ())]]),
             Query(["e1"], [[Product(-1.0, (ident("y"),)), Product(4.0, ())]]),
             Query([], [[Product(1.0, (Factor(F_LE, "d1", 0.25),))], [Product(1.0, (Factor(F_GT, "x1", 0.0),))]])]
    gpu, info = run_gpu(db, batch, info=True)
    assert info["fast_path"]["kind"] == "rt"
    assert_parity(gpu, oracle.evaluate(db, batch), batch)


def test_rt_counts_only_batch():
    db = rt_db(4, 10_000, dyadic=False)
    batch = [Query([], [[Product(1.0, (Factor(F_LE, "x2", t),))] for t in (-1.0, 0.0, 1.0)]),
             Query(["g1"], [[Product(1.0, ())]])]
    gpu, info = run_gpu(db, batch, info=True)
    assert info["fast_path"]["kind"] == "rt"
    assert_parity(gpu, oracle.evaluate(db, batch), batch)


@pytest.mark.parametrize("s", [0.0, 2.0])
def test_rt_skews(s):
    db = rt_db(5, 40_000, s=s)
    batch = c3_like(db, synth.thresholds_c3()[::3], ["x1", "d3"], ["g1", "g3", "c1"])
    assert_parity(run_gpu(db, batch), oracle.evaluate(db, batch), batch)


def test_rt_config3_small_matches_generic(monkeypatch):
    w = synth.config3(fact_rows=60_000, dim_rows=(40, 300, 2000))
    g1, i1 = run_gpu(w.db, w.batch, info=True)
    assert i1["fast_path"]["kind"] == "rt"
    assert_parity(g1, oracle.evaluate(w.db, w.batch), w.batch)
    monkeypatch.setenv("LMFAO_GENERIC_ONLY", "1")
    g2 = run_gpu(w.db, w.batch)
    for (k1, v1, c1), (k2, v2, c2) in zip(g1, g2):
        assert np.array_equal(k1, k2) and np.array_equal(c1, c2)
        assert np.allclose(v1, v2, rtol=1e-11, atol=1e-9)


@pytest.mark.parametrize("nparts", [2, 3])
def test_rt_sharded_partials(nparts):
    w = synth.config3(fact_rows=20_011, dim_rows=(30, 200, 1500))
    ref = oracle.evaluate(w.db, w.batch)
    parts = [run_gpu(w.db, w.batch, shard=(p, nparts)) for p in range(nparts)]
    q = len(w.batch) - 1  # the scalar predicate query
    assert sum(int(p[q][2][0]) for p in parts) == int(ref[q].counts[0])
    assert np.allclose(sum(p[q][1] for p in parts), ref[q].vals, rtol=1e-9, atol=1e-9)
