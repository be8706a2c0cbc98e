"""Group-bys over the attributes of a root child with a non-unique key (SURVEY.md §8(f)
NEXT-4, "group-bys on non-PK dims"): a root row then joins several rows of the child, so the
query is finished at the child — each product's root side summed per key of the child
(A[k][p], the other children through their views), then Σ over the child's rows of
A[key][p] times the product's child side, into the row's cell ("each aggregate to its own
root").  Parity against the oracle."""
import numpy as np
import pytest

import oracle
import synth
from _parity import assert_parity, run_gpu
from synth import F_GE, F_LE, Factor, Product, Query, ident

pytestmark = pytest.mark.gpu


def m2m_db(seed, n, t_child=False):
    """F(k, d, x, c) with T(k, t, tcat, tval) many rows per k, D(d, dv, dcat) a PK dimension;
    optionally U(u, uv) under T."""
    rng = np.random.default_rng(seed)
    nk = 40
    reps = rng.integers(0, 4, nk)  # 0..3 T rows per key (0: the key dangles)
    tk = np.repeat(np.arange(nk, dtype=np.int32), reps)
    perm = rng.permutation(len(tk))
    T = {"k": tk[perm], "tcat": rng.integers(0, 5, len(tk)).astype(np.int32),
         "tval": rng.standard_normal(len(tk)), "t2": rng.integers(0, 3, len(tk)).astype(np.int32)}
    rels = []
    edges = [("F", "T"), ("F", "D")]
    if t_child:
        T["u"] = rng.integers(0, 7, len(tk)).astype(np.int32)
        rels.append(synth.Relation("U", {"u": np.arange(7, dtype=np.int32), "uv": rng.standard_normal(7)}))
        edges.append(("T", "U"))
    D = {"d": np.arange(30, dtype=np.int32), "dv": rng.standard_normal(30), "dcat": rng.integers(0, 4, 30).astype(np.int32)}
    F = {"k": rng.integers(0, nk, n).astype(np.int32), "d": rng.integers(0, 30, n).astype(np.int32),
         "x": rng.standard_normal(n), "c": rng.integers(0, 6, n).astype(np.int32)}
    return synth.Database([synth.Relation("F", F), synth.Relation("T", T), synth.Relation("D", D)] + rels, "F", edges)


def batch(t_child=False):
    P = Product
    qs = [Query(["tcat"], [[P(1.0, ())], [P(1.0, (ident("x"),))], [P(2.0, (ident("tval"),)), P(-1.0, ())],
                           [P(1.0, (ident("x"), ident("tval"), ident("dv")))],
                           [P(1.0, (Factor(F_GE, "x", 0.0), Factor(F_LE, "tval", 0.5)))]]),
          Query(["tcat", "t2"], [[P(1.0, (ident("dv"),))], [P(3.0, ())]]),
          Query(["c"], [[P(1.0, (ident("tval"),))]]),           # root group-by: the fused scan
          Query([], [[P(1.0, (ident("x"), ident("tval")))], [P(1.0, ())]])]
    if t_child:
        qs.append(Query(["t2"], [[P(1.0, (ident("uv"),))], [P(1.0, (ident("uv"), ident("x")))]]))
    return qs


@pytest.mark.parametrize("n", [1, 31, 2_000, 30_000])
def test_groupby_non_unique_child(n):
    db = m2m_db(1, n)
    b = batch()
    assert_parity(run_gpu(db, b), oracle.evaluate(db, b), b)


@pytest.mark.parametrize("seed", [2, 3])
def test_groupby_non_unique_child_with_grandchild(seed):
    db = m2m_db(seed, 20_000, t_child=True)
    b = batch(True)
    assert_parity(run_gpu(db, b), oracle.evaluate(db, b), b)


def test_mixed_group_by_is_rejected():
    from paper_1906_08687_b200 import lmfao
    db = m2m_db(4, 100)
    with pytest.raises(lmfao.LmfaoError) as ei:
        run_gpu(db, [Query(["tcat", "c"], [[Product(1.0, ())]])])
    assert ei.value.name == "LMFAO_ERR_UNSUPPORTED"


def test_sharded_partials():
    db = m2m_db(5, 9_001)
    b = batch()[:2]
    ref = oracle.evaluate(db, b)
    parts = [run_gpu(db, b, shard=(p, 3)) for p in range(3)]
    for qi in range(2):
        tot = {}
        for p in parts:
            k, v, c = p[qi]
            for r in range(len(c)):
                e = tot.setdefault(tuple(k[r]), [0, np.zeros(v.shape[1])])
                e[0] += int(c[r])
                e[1] += v[r]
        assert len(tot) == len(ref[qi].counts)
        for r in range(len(ref[qi].counts)):
            cnt, vals = tot[tuple(ref[qi].keys[r])]
            assert cnt == int(ref[qi].counts[r]) and np.allclose(vals, ref[qi].vals[r], rtol=1e-9, atol=1e-9)
