"""Parity of the specialised covariance (Gram) path — DMMA tiles + run-level
factorisation + dimension-side finishing — against the oracle, over every
template shape (NB row tiles, NS shallower featured levels, NTS tiles per
shallower level), key skews that make runs long or short, featureless dims,
coefficients and sums of products."""
import numpy as np
import pytest

import oracle
import synth
from _parity import assert_parity, run_gpu
from synth import Factor, Product, Query, ident

pytestmark = pytest.mark.gpu


def star(seed, n, nF, dim_feats, dim_rows, s=1.1):
    rng = np.random.default_rng(seed)
    F = {}
    dims = []
    for r, (nf, nr) in enumerate(zip(dim_feats, dim_rows), start=1):
        keys = synth.distinct_keys(synth._rng(seed, "D", r), nr)
        cols = {f"k{r}": keys}
        for j in range(nf):
            cols[f"d{r}_{j}"] = rng.standard_normal(nr)
        dims.append(synth.Relation(f"D{r}", cols))
        F[f"k{r}"] = synth.zipf_fk(seed, "F", f"k{r}", keys, s, n)
    for j in range(nF):
        F[f"x{j}"] = rng.standard_normal(n)
    db = synth.Database([synth.Relation("F", F)] + dims, "F", [("F", d.name) for d in dims])
    feats = [f"x{j}" for j in range(nF)] + [f"d{r}_{j}" for r, nf in enumerate(dim_feats, 1) for j in range(nf)]
    return db, feats


CASES = [
    # (nF, dim feature counts, dim rows) -> (NB, NS, NTS)
    (3, [1, 2], [50, 200]),                  # C1 shape: NB=1, NS=1
    (8, [10, 10, 10], [40, 300, 2000]),      # C2 shape: NB=3, NS=2, NTS=2
    (8, [10], [500]),                        # NS=0
    (5, [3, 12], [30, 700]),                 # NS=1, NTS=1 (A has 3)
    (5, [12, 3], [30, 700]),                 # NS=1, NTS=2 (A has 12)
    (2, [16, 16, 7], [20, 100, 900]),        # NS=2, NTS=2, NB=2
    (1, [2, 2, 2], [5, 7, 11]),              # tiny domains: very long runs
    (8, [4, 0, 6, 0], [30, 60, 600, 5000]),  # featureless dims interleaved in the sort order
    (0, [3, 4], [50, 400]),                  # no fact features
    (8, [0, 4, 4, 4], [30, 100, 1000, 5000]),  # a featureless dim sorts first: B runs nest in its runs
]


FAST = ("cov", "gram")


@pytest.fixture(params=["cov", "cov_cold", "gram"])
def kernel(request, monkeypatch):
    """Run each case through the compile-time-specialised k_cov kernel (cov.cu) — as planned,
    and with LMFAO_COV_COLD_ALL=1, which sends every block down the per-row level-A path
    (exact by linearity) — and, with LMFAO_NO_COV=1, through the general gram.cu kernel."""
    if request.param == "gram":
        monkeypatch.setenv("LMFAO_NO_COV", "1")
    if request.param == "cov_cold":
        monkeypatch.setenv("LMFAO_COV_COLD_ALL", "1")
        return "cov"
    return request.param


@pytest.mark.parametrize("case", range(len(CASES)))
def test_gram_shapes(case, kernel):
    nF, df, dr = CASES[case]
    db, feats = star(case, 30_011 + 7 * case, nF, df, dr)
    batch = [synth.covar_batch(feats)]
    gpu, info = run_gpu(db, batch, info=True)
    fits_cov = nF <= 8 and max(df) <= 10 and sum(1 for f in df if f) <= 3
    want = "cov" if kernel == "cov" and fits_cov else "gram"
    assert info["fast_path"] and info["fast_path"]["kind"] == want, info
    assert_parity(gpu, oracle.evaluate(db, batch), batch)


def test_gram_coefficients_sums_and_repeated_factors(kernel):
    db, feats = star(11, 20_003, 4, [3, 5], [30, 300])
    x0, x1, a, b = "x0", "x1", "d1_0", "d2_4"
    udafs = [
        [Product(2.0, (ident(x0), ident(a))), Product(-3.0, (ident(x1),)), Product(0.5, ())],
        [Product(1.0, (ident(a), ident(a))), Product(1.0, (ident(b), ident(a)))],
        [Product(1.0, (Factor(synth.F_CONST, None, 4.0), ident(x0), ident(x0)))],
        [Product(1.0, (ident(b),)), Product(1.0, (ident(b), ident(b)))],
        [],
    ]
    batch = [Query([], udafs), synth.covar_batch(feats[:3])]
    gpu, info = run_gpu(db, batch, info=True)
    assert info["fast_path"]["kind"] == kernel
    assert_parity(gpu, oracle.evaluate(db, batch), batch)


def test_gram_uniform_and_extreme_skew(kernel):
    for s in (0.0, 2.5):
        db, feats = star(21, 25_000, 6, [4, 4, 4], [30, 200, 3000], s=s)
        batch = [synth.covar_batch(feats)]
        assert_parity(run_gpu(db, batch), oracle.evaluate(db, batch), batch)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 7, 33, 129, 511, 512, 513, 1001, 5000])
def test_gram_tiny_and_ragged_row_counts(n, kernel):
    db, feats = star(31, n, 8, [10, 10, 10], [7, 9, 13])
    batch = [synth.covar_batch(feats)]
    assert_parity(run_gpu(db, batch), oracle.evaluate(db, batch), batch)


def test_gram_matches_generic_path(monkeypatch):
    w = synth.config2(fact_rows=80_000, dim_rows=(40, 300, 2000))
    g1, i1 = run_gpu(w.db, w.batch, info=True)
    monkeypatch.setenv("LMFAO_GENERIC_ONLY", "1")
    g2, i2 = run_gpu(w.db, w.batch, info=True)
    assert i1["fast_path"]["kind"] in FAST and i2["fast_path"] is None
    assert np.array_equal(g1[0][2], g2[0][2])
    assert np.allclose(g1[0][1], g2[0][1], rtol=1e-11, atol=1e-9)


@pytest.mark.parametrize("cube", [True, False])
def test_config5_covariance_uses_gram_with_cube(kernel, cube, monkeypatch):
    """C5: the covariance scan next to the cube path (cube.cu), or next to the generic group scan."""
    if not cube:
        monkeypatch.setenv("LMFAO_NO_CUBE", "1")
    w = synth.config5(fact_rows=30_011, dim_rows=(40, 300, 2000, 9000), cube_doms=(7, 30, 100))
    gpu, info = run_gpu(w.db, w.batch, info=True)
    fp = info["fast_path"]
    if cube:
        assert fp["kind"] == "combo" and fp["scalar"]["kind"] == kernel and fp["groups"]["kind"] == "cube", fp
    else:
        assert fp["kind"] == kernel, fp
    assert_parity(gpu, oracle.evaluate(w.db, w.batch), w.batch)


@pytest.mark.parametrize("nparts", [2, 5])
def test_gram_sharded_partials(nparts, kernel):
    w = synth.config2(fact_rows=40_007, dim_rows=(30, 200, 1500))
    ref = oracle.evaluate(w.db, w.batch)[0]
    parts = [run_gpu(w.db, w.batch, shard=(p, nparts))[0] for p in range(nparts)]
    assert sum(int(p[2][0]) for p in parts) == int(ref.counts[0])
    assert np.allclose(sum(p[1] for p in parts), ref.vals, rtol=1e-9, atol=1e-9)
