"""NEXT-2 batches: categorical covariance — one-hot categorical features as
group-bys, Covar(X_j; X_k) = SUM(X_j) GROUP BY X_k and Covar(X_j, X_k; 1) = COUNT GROUP BY
(X_j, X_k) — and degree-2 polynomial regression aggregates, products of
up to four identity factors.  Parity against the oracle on whatever path the
planner picks (the interpreted path covers every shape)."""
import itertools

import numpy as np
import pytest

import oracle
import synth
from _parity import assert_parity, run_gpu
from synth import Product, Query, ident

pytestmark = pytest.mark.gpu


def cat_db(seed, n):
    rng = np.random.default_rng(seed)
    w = synth.config2(seed=seed, fact_rows=n, dim_rows=(30, 200, 1500))
    db = w.db
    F = db.rel("F")
    F.cols["cf"] = rng.integers(0, 6, n).astype(np.int32)
    for r, d in ((1, 4), (3, 9)):
        R = db.rel(f"D{r}")
        R.cols[f"cat{r}"] = rng.integers(0, d, R.nrows).astype(np.int32)
    return db


def categorical_covar_batch(conts, cats):
    qs = [synth.covar_batch(conts)]
    for k in cats:  # Covar(X_j; X_k): SUM(X_j) and COUNT per category of X_k
        qs.append(Query([k], [[Product(1.0, ())]] + [[Product(1.0, (ident(j),))] for j in conts]))
    for a, b in itertools.combinations(cats, 2):  # Covar(X_j, X_k; 1)
        qs.append(Query([a, b], [[Product(1.0, ())]]))
    return qs


def poly2_batch(feats):
    """Σ of every monomial of degree <= 4 in the features (the Gram of degree-2 monomials)."""
    mons = [()] + [(f,) for f in feats] + list(itertools.combinations_with_replacement(feats, 2))
    udafs = []
    for i, m1 in enumerate(mons):
        for m2 in mons[i:]:
            udafs.append([Product(1.0, tuple(ident(a) for a in m1 + m2))])
    return [Query([], udafs)]


@pytest.mark.parametrize("n", [1, 777, 20_000])
def test_categorical_covariance(n):
    db = cat_db(1, n)
    batch = categorical_covar_batch(["x1", "x2", "d1_1", "d3_2"], ["cf", "cat1", "cat3"])
    assert_parity(run_gpu(db, batch), oracle.evaluate(db, batch), batch)


@pytest.mark.parametrize("path", ["poly", "generic"])
@pytest.mark.parametrize("n", [1, 5_000, 40_013])
def test_degree2_polynomial(n, path, monkeypatch):
    """poly: the Gram of the degree-2 monomials as FP64 DMMA tiles (poly.cu); generic: the
    interpreted scan (LMFAO_NO_POLY=1)."""
    if path == "generic":
        monkeypatch.setenv("LMFAO_NO_POLY", "1")
    db = cat_db(2, n)
    batch = poly2_batch(["x1", "d2_1", "d3_3"])  # monomials over the root and two dimensions
    assert sum(len(q.udafs) for q in batch) == 55
    gpu, info = run_gpu(db, batch, info=True)
    assert (info["fast_path"] or {}).get("kind") == (path if path == "poly" else None), info["fast_path"]
    assert_parity(gpu, oracle.evaluate(db, batch), batch)


@pytest.mark.parametrize("feats", [["x1", "x2", "d1_1", "d3_1"], ["x1", "x2", "x3", "d1_2", "d2_2", "d3_4"]])
def test_degree2_polynomial_more_features_and_coefficients(feats):
    """Up to 24 halves (six features: 1 + 6 + 21 = 28 monomials would not fit, so the planner
    splits products over the halves it has), sums of products with coefficients, constants."""
    db = cat_db(3, 30_011)
    batch = poly2_batch(feats[:4])
    P, I = Product, ident
    f = feats
    batch.append(Query([], [[P(2.0, (I(f[0]), I(f[1]), I(f[2]))), P(-1.5, (I(f[-1]),)), P(0.25, ())],
                            [P(1.0, (I(f[-1]), I(f[-1]), I(f[-2]), I(f[-3])))], []]))
    gpu, info = run_gpu(db, batch, info=True)
    assert_parity(gpu, oracle.evaluate(db, batch), batch)


@pytest.mark.parametrize("n", [1, 31, 4097, 60_013])
def test_fact_only_covariance_on_the_gram_kernel(n):
    """A relation without children (the fact-only Gram of SURVEY §8(d)): cov.cu and gram.cu need
    root children, so poly.cu's Gram of halves [1, x_1..x_8] takes it (45 distinct entries)."""
    rng = np.random.default_rng(n)
    cols = {f"x{j}": rng.standard_normal(n) for j in range(7)}
    cols["i"] = rng.integers(-5, 6, n).astype(np.int32)  # eight features: poly.cu's limit
    db = synth.Database([synth.Relation("F", cols)], "F", [])
    batch = [synth.covar_batch(list(cols))]
    gpu, info = run_gpu(db, batch, info=True)
    assert info["fast_path"]["kind"] == "poly", info["fast_path"]
    assert_parity(gpu, oracle.evaluate(db, batch), batch)
