"""Regression-tree node batches with a path condition (§3
"Regression trees" P:528-555: a node's aggregates carry α = Π of Kronecker deltas along the
path from the root of the tree): rt.cu takes the predicates every product shares as a per-row
filter (root attributes directly, dimension attributes through the foreign keys), the sums
under the filter, and the join multiplicities (group presence, counts) from an unconditioned
pass.  Parity against the oracle, which evaluates the products as written."""
import numpy as np
import pytest

import oracle
import synth
from _parity import assert_parity, run_gpu
from synth import F_EQ, F_GE, F_GT, F_LE, F_LT, F_NE, Factor, Product, Query, ident

pytestmark = pytest.mark.gpu


def rt_db(seed, n, dim_rows=(30, 200, 1500), s=1.1):
    rng = np.random.default_rng(seed)
    F, dims = {}, []
    for r, nr in enumerate(dim_rows, start=1):
        keys = synth.distinct_keys(synth._rng(seed, "RTP", r), nr)
        dims.append(synth.Relation(f"D{r}", {f"k{r}": keys, f"d{r}": np.round(rng.standard_normal(nr) * 4) / 4,
                                              f"e{r}": rng.integers(-3, 4, nr).astype(np.int32),
                                              f"g{r}": rng.integers(0, 5 + 7 * r, nr).astype(np.int32)}))
        F[f"k{r}"] = synth.zipf_fk(seed, "F", f"k{r}", keys, s, n)
    F["x1"] = np.round(rng.standard_normal(n) * 8) / 8
    F["x2"] = rng.standard_normal(n)
    F["i1"] = rng.integers(-5, 6, n).astype(np.int32)
    F["c1"] = rng.integers(0, 9, n).astype(np.int32)
    F["c2"] = rng.integers(0, 600, n).astype(np.int32)
    F["y"] = rng.standard_normal(n)
    return synth.Database([synth.Relation("F", F)] + dims, "F", [("F", d.name) for d in dims])


def node_batch(path, splits, cats, ts=(-1.0, -0.25, 0.0, 0.5, 1.25)):
    """A CART node: totals φ·y^p, split aggregates φ·1[A op t]·y^p, categorical group-bys."""
    def prods(extra, p):
        return [Product(1.0, tuple(path) + tuple(extra) + (ident("y"),) * p)]
    udafs = [prods((), p) for p in range(3)]
    for a, op in splits:
        for t in ts:
            for p in range(3):
                udafs.append(prods((Factor(op, a, t),), p))
    qs = [Query([], udafs)]
    for cat in cats:
        qs.append(Query([cat], [prods((), p) for p in range(3)]))
    return qs


PATH = [Factor(F_GE, "x1", -0.5), Factor(F_LE, "d2", 0.25), Factor(F_GT, "e3", -2)]
SPLITS = [("x2", F_LE), ("x1", F_GT), ("i1", F_LT), ("d1", F_GE), ("e2", F_EQ), ("d3", F_NE)]


@pytest.mark.parametrize("n", [1, 33, 5_000, 40_011])
def test_node_with_path(n):
    db = rt_db(1, n)
    batch = node_batch(PATH, SPLITS, ["c1", "c2", "g1", "g3"])
    gpu, info = run_gpu(db, batch, info=True)
    fp = info["fast_path"]
    assert fp["kind"] == "rt" and fp["path_preds"] == 3, fp
    assert_parity(gpu, oracle.evaluate(db, batch), batch)


@pytest.mark.parametrize("depth", [1, 2, 4])
def test_path_depths_match_generic(depth, monkeypatch):
    db = rt_db(2, 30_000)
    path = [Factor(F_GT, "x2", -1.0), Factor(F_LE, "d1", 0.5), Factor(F_NE, "i1", 0), Factor(F_GE, "e2", -1)][:depth]
    batch = node_batch(path, SPLITS[:3], ["g2", "c1"])
    g1, info = run_gpu(db, batch, info=True)
    assert info["fast_path"]["path_preds"] == depth
    assert_parity(g1, oracle.evaluate(db, batch), batch)
    monkeypatch.setenv("LMFAO_GENERIC_ONLY", "1")
    g2 = run_gpu(db, batch)
    for (k1, v1, c1), (k2, v2, c2) in zip(g1, g2):
        assert np.array_equal(k1, k2) and np.array_equal(c1, c2)
        assert np.allclose(v1, v2, rtol=1e-11, atol=1e-9)


def test_path_no_row_passes():
    """An empty node: every sum is 0, the group-bys still list every present group with its
    join multiplicity (reading R2)."""
    db = rt_db(3, 8_000)
    batch = node_batch([Factor(F_GT, "x2", 100.0)], SPLITS[:2], ["c1", "g2"])
    gpu = run_gpu(db, batch)
    ref = oracle.evaluate(db, batch)
    assert_parity(gpu, ref, batch)
    assert not np.any(gpu[0][1]) and int(gpu[0][2][0]) == 8_000
    assert len(gpu[1][2]) == len(ref[1].counts) > 0


def test_path_only_scalar_and_repeated_predicate():
    db = rt_db(4, 12_000)
    path = [Factor(F_LT, "d3", 0.0)]
    udafs = [[Product(1.0, tuple(path))], [Product(2.0, tuple(path) + (ident("y"),))],
             [Product(1.0, tuple(path) + (Factor(F_LT, "d3", 0.0),))],   # the path predicate twice
             [Product(1.0, tuple(path) + (Factor(F_GE, "x1", 0.0),)), Product(-1.0, tuple(path))]]
    batch = [Query([], udafs)]
    gpu, info = run_gpu(db, batch, info=True)
    assert info["fast_path"]["kind"] == "rt" and info["fast_path"]["path_preds"] == 1
    assert_parity(gpu, oracle.evaluate(db, batch), batch)


def test_path_sharded_partials():
    db = rt_db(5, 20_011)
    batch = node_batch(PATH[:2], SPLITS[:2], [])
    ref = oracle.evaluate(db, batch)[0]
    parts = [run_gpu(db, batch, shard=(p, 3))[0] for p in range(3)]
    assert sum(int(p[2][0]) for p in parts) == int(ref.counts[0])
    assert np.allclose(sum(p[1] for p in parts), ref.vals, rtol=1e-9, atol=1e-9)


def ct_batch(path, cls, splits, ts=(-0.5, 0.0, 0.75)):
    """A classification node: CT(X; α) and CT(X; α·1[A op t]) for the class X, plus
    CT(α); here also y-weighted variants and the node's regression totals."""
    P = tuple(path)
    qs = [Query([cls], [[Product(1.0, P)], [Product(1.0, P + (ident("y"),))]])]
    for a, op in splits:
        qs.append(Query([cls], [[Product(1.0, P + (Factor(op, a, t),))] for t in ts] +
                        [[Product(0.5, P + (Factor(op, a, ts[0]), ident("y")))]]))
    qs.append(Query([], [[Product(1.0, P)], [Product(1.0, P + (Factor(F_LE, "x2", 0.0),))]]))
    return qs


@pytest.mark.parametrize("cls", ["c1", "g1"])
@pytest.mark.parametrize("with_path", [False, True])
def test_classification_node(cls, with_path):
    db = rt_db(6, 25_000)
    path = PATH[:2] if with_path else []
    batch = ct_batch(path, cls, [("x2", F_LE), ("d3", F_GT), ("i1", F_EQ), ("e2", F_NE)])
    gpu, info = run_gpu(db, batch, info=True)
    fp = info["fast_path"]
    assert fp["kind"] == "rt" and fp["classes"] > 0 and fp["path_preds"] == len(path), fp
    assert_parity(gpu, oracle.evaluate(db, batch), batch)


@pytest.mark.parametrize("n", [1, 31, 2_049])
def test_classification_node_small(n):
    db = rt_db(7, n)
    batch = ct_batch(PATH, "c1", [("x1", F_GE), ("d1", F_LT)]) + [Query(["g2"], [[Product(1.0, tuple(PATH))]])]
    gpu, info = run_gpu(db, batch, info=True)
    assert info["fast_path"]["kind"] == "rt", info["fast_path"]
    assert_parity(gpu, oracle.evaluate(db, batch), batch)


def test_path_with_set_inclusion():
    """Categorical splits on the path (LMFAO_F_IN): root and dimension categoricals."""
    from synth import F_IN
    db = rt_db(8, 20_000)
    path = [Factor(F_IN, "c1", float((1 << 0) | (1 << 3) | (1 << 4) | (1 << 8))),
            Factor(F_IN, "g2", float(sum(1 << v for v in range(0, 19, 2)))), Factor(F_GE, "x2", -1.0)]
    batch = node_batch(path, SPLITS[:4], ["g1", "c2"])
    gpu, info = run_gpu(db, batch, info=True)
    assert info["fast_path"]["kind"] == "rt" and info["fast_path"]["path_preds"] == 3, info["fast_path"]
    assert_parity(gpu, oracle.evaluate(db, batch), batch)


def test_set_inclusion_in_products_interpreted():
    """LMFAO_F_IN inside products the histogram path does not take: the interpreted scan."""
    from synth import F_IN
    db = rt_db(9, 6_000)
    m = float((1 << 1) | (1 << 2) | (1 << 52))
    batch = [Query(["c1"], [[Product(1.0, (Factor(F_IN, "g3", m),))], [Product(1.0, (Factor(F_IN, "e1", m), ident("x2")))]]),
             Query([], [[Product(1.0, (Factor(F_IN, "i1", m), ident("y"), ident("x1")))]])]
    assert_parity(run_gpu(db, batch), oracle.evaluate(db, batch), batch)


def test_set_condition_rebinds_the_path_without_replanning():
    """Dynamic functions: a batch planned under path condition φ1, rebound
    to φ2, φ3 (root, dimension and set-inclusion predicates, a different number of them, and
    the empty condition) by lmfao_set_condition, equals the oracle of the batch written with φ2,
    φ3 in place of φ1 — counts of the group-by queries included (join multiplicities)."""
    from paper_1906_08687_b200 import lmfao
    w = synth.config3(fact_rows=40_011, dim_rows=(30, 200, 1500))
    F = synth.Factor
    phi1 = [F(synth.F_GE, "y", float("-inf"))]
    phi2 = [F(synth.F_LE, "x1", 0.25), F(synth.F_GT, "d2_3", -0.5)]
    phi3 = [F(synth.F_GT, "d1_2", 0.0), F(synth.F_IN, "c1", float((1 << 2) | (1 << 5) | (1 << 7))),
            F(synth.F_LE, "d3_1", 1.0)]

    def batch(phi):
        y = synth.ident("y")
        u = [[synth.Product(1.0, tuple(phi) + (y,) * p)] for p in range(3)]
        for a in ("x2", "d1_1", "d3_4"):
            for t in (-0.5, 0.0, 0.75):
                u += [[synth.Product(1.0, tuple(phi) + (F(synth.F_LE, a, t),) + (y,) * p)] for p in range(3)]
        g = [synth.Query([x], [[synth.Product(1.0, tuple(phi) + (y,) * p)] for p in range(3)]) for x in ("c1", "c3")]
        return [synth.Query([], u)] + g

    e = lmfao.Engine()
    try:
        qids = lmfao.load(e, w.db, batch(phi1))
        e.plan()
        assert e.plan_info()["fast_path"]["kind"] == "rt"
        for phi in (phi2, phi3, [], phi2):
            e.set_condition(phi)
            e.run()
            got = [e.fetch(q) for q in qids]
            assert_parity(got, oracle.evaluate(w.db, batch(phi)), batch(phi))
    finally:
        e.close()
