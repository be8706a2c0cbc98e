"""Parity of the cube path (cube.cu, §8 row (e)(iii)): group-by batches of SUMs linear in
root measures over attributes of the root and its primary-key children, cells updated once
per run at the level of their deepest group-by attribute.  Covers the C5 shape (data cube
next to a covariance batch: combined with cov.cu), group-by attributes on the root (level-R
runs), several attributes of one dimension, int32 and fp64 measures, linear combinations
with constants, constant (COUNT-like) UDAFs, ragged row counts around the 32-row block and
the 2048-row work-chunk boundaries, and agreement with the generic scan."""
import numpy as np
import pytest

import oracle
import synth
from _parity import assert_parity, run_gpu
from synth import Factor, Product, Query, ident

pytestmark = pytest.mark.gpu


def c5_small(n, seed=0):
    return synth.config5(seed=seed, fact_rows=n, dim_rows=(20, 150, 1_200, 5_000), cube_doms=(5, 30, 200))


def cube_db(seed, n, dim_rows=(40, 300, 2_000)):
    rng = np.random.default_rng(seed)
    F, dims = {}, []
    for r, nr in enumerate(dim_rows, start=1):
        keys = synth.distinct_keys(synth._rng(seed, "CB", r), nr)
        dims.append(synth.Relation(f"D{r}", {f"k{r}": keys,
                                              f"a{r}": rng.integers(0, 4 + 3 * r, nr).astype(np.int32),
                                              f"b{r}": rng.integers(-2, 3, nr).astype(np.int32),
                                              f"x{r}": rng.standard_normal(nr)}))
        F[f"k{r}"] = synth.zipf_fk(seed, "F", f"k{r}", keys, 1.1, n)
    F["g"] = rng.integers(0, 6, n).astype(np.int32)
    F["h"] = rng.integers(0, 3, n).astype(np.int32)
    F["m1"] = rng.random(n) * 100
    F["m2"] = rng.standard_normal(n)
    F["i1"] = rng.integers(-50, 50, n).astype(np.int32)
    return synth.Database([synth.Relation("F", F)] + dims, "F", [("F", d.name) for d in dims])


def S(*terms):  # UDAF = Σ coeff * attr (attr None: constant)
    return [Product(c, (ident(a),) if a else ()) for c, a in terms]


def rich_batch():
    return [Query(["a1"], [S((1, "m1")), S((1, "m2"))]),
            Query(["a3"], [S((1, "m1")), S((2, "m2"), (-1, "i1"), (3, None))]),
            Query(["a1", "a2", "a3"], [S((1, "m1")), S((1, None))]),
            Query(["a2", "b2"], [S((1, "i1"))]),
            Query(["g"], [S((1, "m2"))]),
            Query(["a1", "g", "h"], [S((1, "m1")), S((0.5, "i1"))]),
            Query(["h", "a3"], [S((1, None)), S((1, "m2"))]),
            Query([], [S((1, "m1")), S((1, None))])]


def test_c5_shape_combo():
    w = c5_small(60_000)
    gpu, info = run_gpu(w.db, w.batch, info=True)
    fp = info["fast_path"]
    assert fp["kind"] == "combo" and fp["groups"]["kind"] == "cube" and fp["scalar"]["kind"] == "cov", fp
    assert_parity(gpu, oracle.evaluate(w.db, w.batch), w.batch)


@pytest.mark.parametrize("n", [1, 31, 33, 2047, 2048, 2049, 4097, 20_000])
def test_cube_ragged(n):
    db = cube_db(1, n)
    batch = rich_batch()
    gpu, info = run_gpu(db, batch, info=True)
    assert info["fast_path"]["groups"]["kind"] == "cube", info["fast_path"]
    assert_parity(gpu, oracle.evaluate(db, batch), batch)


@pytest.mark.parametrize("small", ["1", "0"])
def test_cube_small_tables_in_shared_memory(small, monkeypatch):
    """Dense cuboids of at most 1024 values (cells x (UDAFs + 1)) accumulate in a per-CTA copy in
    shared memory, flushed once (LMFAO_CUBE_SMALL=0: global REDs throughout); a root group-by
    attribute makes nearly every row a run end, the case the copies are for."""
    db = cube_db(12, 30_011)
    monkeypatch.setenv("LMFAO_CUBE_SMALL", small)
    batch = rich_batch()
    gpu, info = run_gpu(db, batch, info=True, runs=2)
    assert info["fast_path"]["groups"]["kind"] == "cube", info["fast_path"]
    assert_parity(gpu, oracle.evaluate(db, batch), batch)


@pytest.mark.parametrize("s", [0.0, 2.5])
def test_cube_skew_matches_generic(s, monkeypatch):
    db = cube_db(2, 50_000)
    for r in (1, 2, 3):
        d = db.rel(f"D{r}")
        db.rel("F").cols[f"k{r}"] = synth.zipf_fk(7, "F", f"k{r}", d.cols[f"k{r}"], s, 50_000)
    batch = rich_batch()
    g1 = run_gpu(db, batch)
    assert_parity(g1, oracle.evaluate(db, batch), batch)
    monkeypatch.setenv("LMFAO_NO_CUBE", "1")
    g2 = run_gpu(db, batch)
    for (k1, v1, c1), (k2, v2, c2) in zip(g1, g2):
        assert np.array_equal(k1, k2) and np.array_equal(c1, c2)
        assert np.allclose(v1, v2, rtol=1e-11, atol=1e-9)


def test_cube_sharded_partials():
    db = cube_db(3, 30_011)
    batch = rich_batch()[:4]
    ref = oracle.evaluate(db, batch)
    parts = [run_gpu(db, batch, shard=(p, 3)) for p in range(3)]
    for qi, q in enumerate(batch):  # every part's groups are a subset; their sums add up
        tot = {}
        for p in parts:
            k, v, c = p[qi]
            for row in range(len(c)):
                key = tuple(k[row])
                cv = tot.setdefault(key, [0, np.zeros(v.shape[1])])
                cv[0] += int(c[row])
                cv[1] += v[row]
        assert len(tot) == len(ref[qi].counts)
        for row in range(len(ref[qi].counts)):
            cnt, vals = tot[tuple(ref[qi].keys[row])]
            assert cnt == int(ref[qi].counts[row])
            assert np.allclose(vals, ref[qi].vals[row], rtol=1e-9, atol=1e-9)


def test_cube_declines_non_linear():
    db = cube_db(4, 5_000)
    batch = [Query(["a1"], [[Product(1.0, (ident("m1"), ident("m2")))]])]  # a product of two measures
    gpu, info = run_gpu(db, batch, info=True)
    assert info["fast_path"] is None or info["fast_path"].get("kind") != "combo"
    assert_parity(gpu, oracle.evaluate(db, batch), batch)


@pytest.mark.parametrize("n", [1, 2049, 30_000])
def test_cube_sparse_records(n, monkeypatch):
    """Cuboids above the dense-table threshold: sorted run records reduced after the scan
    (threshold lowered so the small test cube takes that path); equal to the dense path."""
    db = cube_db(5, n)
    batch = rich_batch()
    monkeypatch.setenv("LMFAO_CUBE_SPARSE_CELLS", "20")
    g1, info = run_gpu(db, batch, info=True, runs=2)
    assert info["fast_path"]["groups"]["sparse"] >= 1, info["fast_path"]
    assert_parity(g1, oracle.evaluate(db, batch), batch)
    monkeypatch.setenv("LMFAO_CUBE_SPARSE_CELLS", str(1 << 40))
    g2, info2 = run_gpu(db, batch, info=True)
    assert info2["fast_path"]["groups"]["sparse"] == 0
    for (k1, v1, c1), (k2, v2, c2) in zip(g1, g2):
        assert np.array_equal(k1, k2) and np.array_equal(c1, c2)
        assert np.allclose(v1, v2, rtol=1e-11, atol=1e-9)


@pytest.mark.parametrize("n", [1, 4097, 40_000])
def test_cube_rollups_from_sparse(n, monkeypatch):
    """Every cuboid over a subset of a sparse cuboid's attributes is rolled up from its sorted
    groups: prefix subsets by segmented warp sums, others merged per tile from the segments of
    the dropped attributes (k_merge_rollup, opt-in: LMFAO_CUBE_MERGE=1; LMFAO_CUBE_MERGE_MIN
    lowers its size threshold) or by per-group REDs, the smaller ones from those tables; the scan keeps only the sparse
    level (k_cube_rec).  All three rollup routes against the oracle."""
    db = cube_db(11, n)
    batch = [Query(["a1", "a2", "a3"], [S((1, "m1")), S((1, "m2"), (2, None))]),
             Query(["a2", "a3"], [S((1, "m1")), S((1, "m2"), (2, None))]),
             Query(["a1", "a3"], [S((1, "m1")), S((1, "m2"), (2, None))]),
             Query(["a3", "a1"], [S((1, "m1")), S((1, "m2"), (2, None))]),
             Query(["a1", "a2"], [S((1, "m1")), S((1, "m2"), (2, None))]),
             Query(["a3"], [S((1, "m1")), S((1, "m2"), (2, None))]),
             Query(["a2"], [S((1, "m2"))]),
             Query([], [S((1, "m1")), S((1, None))])]
    ref = oracle.evaluate(db, batch)
    monkeypatch.setenv("LMFAO_CUBE_SPARSE_CELLS", "500")  # {a1,a2,a3}: 910 cells; the others dense
    for merge, gather in (("1", "0"), ("0", "0"), ("0", "1")):  # merged / RED rollups; records gathered first
        monkeypatch.setenv("LMFAO_CUBE_MERGE", merge)
        monkeypatch.setenv("LMFAO_CUBE_MERGE_MIN", "1")
        monkeypatch.setenv("LMFAO_CUBE_GATHER", gather)
        gpu, info = run_gpu(db, batch, info=True, runs=2)
        g = info["fast_path"]["groups"]
        assert g["sparse"] == 1 and g["scan"] == "records", g
        assert_parity(gpu, ref, batch)


def test_c5_cube_sparse_abc():
    """C5's {A,B,C} cuboid at its full 5·10^8-cell domain takes the sparse path."""
    w = synth.config5(fact_rows=200_000, dim_rows=(1_000, 10_000, 100_000, 1_000_000))
    gpu, info = run_gpu(w.db, w.batch, info=True)
    assert info["fast_path"]["groups"]["sparse"] == 1, info["fast_path"]
    assert_parity(gpu, oracle.evaluate(w.db, w.batch), w.batch)


def test_cube_dimension_measures():
    """Measures owned by primary-key dimensions (Covar(X_j; X_k) with X_j a dimension feature,
    NEXT-2): read through the dense foreign keys."""
    db = cube_db(8, 20_000)
    batch = [Query(["a1"], [S((1, "x2")), S((1, "m1")), S((2, "x3"), (1, None))]),
             Query(["g", "a3"], [S((1, "x1"))]),
             Query(["a2", "b2"], [S((-1, "x3"))])]
    gpu, info = run_gpu(db, batch, info=True)
    assert info["fast_path"]["groups"]["kind"] == "cube", info["fast_path"]
    assert_parity(gpu, oracle.evaluate(db, batch), batch)


def test_cube_many_measures():
    """More measures than one scan carries (8): one scan per group of 8, the counts with the
    first; UDAFs mixing measures of different groups are added in parts."""
    db = cube_db(10, 15_000)
    rng = np.random.default_rng(3)
    F = db.rel("F")
    extra = []
    for j in range(9):
        F.cols[f"z{j}"] = rng.standard_normal(F.nrows)
        extra.append(f"z{j}")
    ms = ["m1", "m2", "i1", "x1", "x2"] + extra  # 14 measures (x* on dimensions)
    batch = [Query(["a1"], [S((1, m)) for m in ms]),
             Query(["g", "a3"], [S((1, "z0"), (2, "z8"), (-1, None)), S((1, "x2"), (1, "m1"))]),
             Query(["a2"], [S((3, "z5"))] + [S((1, None))])]
    gpu, info = run_gpu(db, batch, info=True)
    fp = info["fast_path"]["groups"]
    assert fp["kind"] == "cube" and fp["scans"] == 2 and fp["measures"] == 14, fp
    assert_parity(gpu, oracle.evaluate(db, batch), batch)


@pytest.mark.parametrize("n", [257, 3001, 40_009])  # enough rows for {a1,g,a2}'s ~420 present cells
def test_cube_records_at_the_root_level(n, monkeypatch):
    """k_cube_rec when the sparse cuboid groups by a root attribute (its runs at level R: equal
    keys and equal root codes) and the measures are not all fp64 root columns (the general
    load path), every other cuboid a rollup of it."""
    db = cube_db(13, n)
    sums = [S((1, "m1")), S((1, "i1")), S((2, "m2"), (1, None)), S((1, "x2"))]  # x2: a dimension measure
    batch = [Query(["a1", "g", "a2"], sums), Query(["g"], sums), Query(["a1", "g"], sums),
             Query(["a2"], sums), Query([], sums)]
    monkeypatch.setenv("LMFAO_CUBE_SPARSE_CELLS", "100")
    gpu, info = run_gpu(db, batch, info=True, runs=2)
    g = info["fast_path"]["groups"] if "groups" in info["fast_path"] else info["fast_path"]
    assert g["kind"] == "cube" and g["sparse"] == 1 and g["scan"] == "records", info["fast_path"]
    assert_parity(gpu, oracle.evaluate(db, batch), batch)
