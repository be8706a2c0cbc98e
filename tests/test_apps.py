"""Downstream consumers (paper_1906_08687_b200/apps.py): ridge
regression by BGD over the covar matrix, mutual information and the Chow-Liu tree.  Pinned to
a pandas materialisation of the join (least squares / empirical MI on the joined rows), closed
forms, and brute force over all spanning trees; the GPU test feeds lmfao_fetch results."""
import itertools
import math

import numpy as np
import pandas as pd
import pytest

import oracle
import synth
from paper_1906_08687_b200 import apps


def _join(db):
    frames = {r.name: pd.DataFrame({c: v for c, v in r.cols.items()}) for r in db.relations}
    J = frames[db.root]
    for p, c in db.edges:
        f = frames[c]
        J = J.merge(f, on=[x for x in f.columns if x in J.columns], how="inner")
    return J


def _small_star(seed=0, n=3000):
    w = synth.config2(seed=seed, fact_rows=n, dim_rows=(20, 60, 200))
    feats = w.meta["features"][:5] + ["d1_1", "d3_2"]
    return w.db, feats


@pytest.mark.parametrize("lam", [0.0, 1e-2, 1.0])
def test_ridge_bgd_matches_lstsq_on_materialised_join(lam):
    db, feats = _small_star()
    label = len(feats)  # the last feature is the label; column 0 is the intercept
    res = oracle.evaluate(db, [synth.covar_batch(feats)])[0]
    C = apps.covar_matrix(feats, res.vals[0])
    J = _join(db)
    X = np.concatenate([np.ones((len(J), 1)), J[feats[:-1]].to_numpy()], axis=1)
    y = J[feats[-1]].to_numpy()
    assert np.allclose(C, np.concatenate([X, y[:, None]], axis=1).T @ np.concatenate([X, y[:, None]], axis=1),
                       rtol=1e-10)
    N = len(J)
    exp = np.linalg.solve(X.T @ X / N + lam * np.eye(X.shape[1]), X.T @ y / N)
    theta, it, ok = apps.ridge_bgd(C, label, lam=lam, tol=1e-12)
    assert ok, it
    assert np.allclose(theta, exp, rtol=1e-6, atol=1e-8), (theta, exp)
    assert np.allclose(apps.ridge_closed_form(C, label, lam), exp, rtol=1e-9, atol=1e-12)
    # the objective from C equals the objective on the rows
    J_rows = 0.5 * np.mean((X @ theta - y) ** 2) + 0.5 * lam * theta @ theta
    assert math.isclose(apps.ridge_objective(C, label, theta, lam), J_rows, rel_tol=1e-9)


def test_ridge_gradient_is_the_derivative():
    db, feats = _small_star(1, 800)
    C = apps.covar_matrix(feats, oracle.evaluate(db, [synth.covar_batch(feats)])[0].vals[0])
    rng = np.random.default_rng(0)
    th = rng.standard_normal(len(feats))
    g = apps.ridge_gradient(C, 3, th, 0.1)
    h = 1e-6
    num = np.array([(apps.ridge_objective(C, 3, th + h * e, 0.1) - apps.ridge_objective(C, 3, th - h * e, 0.1)) / (2 * h)
                    for e in np.eye(len(th))])
    assert np.allclose(g, num, rtol=1e-5, atol=1e-7)


def _mi_db(seed=0, n=4000):
    rng = np.random.default_rng(seed)
    keys = np.arange(50, dtype=np.int32)
    D = {"k": keys, "b": rng.integers(0, 4, 50).astype(np.int32), "c": rng.integers(0, 3, 50).astype(np.int32)}
    k = rng.integers(0, 50, n).astype(np.int32)
    a = rng.integers(0, 5, n).astype(np.int32)
    e = ((a + D["b"][k]) % 3).astype(np.int32)  # e depends on a and b: high MI
    return synth.Database([synth.Relation("F", {"k": k, "a": a, "e": e}), synth.Relation("D", D)], "F", [("F", "D")])


def _results(db, batch):
    return [(r.keys, r.vals, r.counts) for r in oracle.evaluate(db, batch)]


def test_mi_matches_empirical_mi_of_the_join():
    db = _mi_db()
    attrs = ["a", "b", "c", "e"]
    M = apps.mi_matrix(attrs, _results(db, synth.mi_batch(attrs)))
    J = _join(db)
    for i, j in itertools.combinations(range(4), 2):
        p = pd.crosstab(J[attrs[i]], J[attrs[j]]).to_numpy() / len(J)
        pi, pj = p.sum(1, keepdims=True), p.sum(0, keepdims=True)
        nz = p > 0
        exp = float((p[nz] * np.log(p[nz] / (pi @ pj)[nz])).sum())
        assert math.isclose(M[i, j], exp, rel_tol=1e-12, abs_tol=1e-15), (attrs[i], attrs[j])
    assert np.all(M >= -1e-15) and np.array_equal(M, M.T)


def test_mi_of_independent_and_identical_attributes():
    # identical attributes: MI = entropy; a constant attribute: MI = 0
    total = 8
    marg = {0: 2, 1: 6}
    pair_same = {(0, 0): 2, (1, 1): 6}
    H = -(0.25 * math.log(0.25) + 0.75 * math.log(0.75))
    assert math.isclose(apps.mutual_information(total, marg, marg, pair_same), H, rel_tol=1e-15)
    assert apps.mutual_information(total, marg, {7: 8}, {(0, 7): 2, (1, 7): 6}) == 0.0


def _brute_max_spanning(M):
    n = M.shape[0]
    best, arg = -1.0, None
    edges = [(i, j) for i in range(n) for j in range(i + 1, n)]
    for sub in itertools.combinations(edges, n - 1):
        parent = list(range(n))

        def find(x):
            while parent[x] != x:
                x = parent[x]
            return x
        ok = True
        for i, j in sub:
            ri, rj = find(i), find(j)
            if ri == rj:
                ok = False
                break
            parent[ri] = rj
        if ok:
            w = sum(M[i, j] for i, j in sub)
            if w > best:
                best, arg = w, set(sub)
    return best, arg


@pytest.mark.parametrize("seed", range(6))
def test_chow_liu_is_a_maximum_spanning_tree(seed):
    rng = np.random.default_rng(seed)
    n = 6
    A = rng.random((n, n))
    M = np.triu(A, 1) + np.triu(A, 1).T
    tree = apps.chow_liu_tree(M)
    best, arg = _brute_max_spanning(M)
    assert len(tree) == n - 1 and math.isclose(sum(M[i, j] for i, j in tree), best, rel_tol=1e-12)
    assert set(tree) == arg


def test_chow_liu_on_mi_of_the_join():
    db = _mi_db(3)
    attrs = ["a", "b", "c", "e"]
    M = apps.mi_matrix(attrs, _results(db, synth.mi_batch(attrs)))
    tree = apps.chow_liu_tree(M)
    assert len(tree) == 3
    assert (0, 3) in tree or (1, 3) in tree  # e = (a + b) mod 3 hangs off a or b


@pytest.mark.gpu
def test_consumers_on_gpu_results():
    from _parity import run_gpu
    db, feats = _small_star(4, 20_000)
    gpu = run_gpu(db, [synth.covar_batch(feats)])
    C = apps.covar_matrix(feats, gpu[0][1][0])
    Cref = apps.covar_matrix(feats, oracle.evaluate(db, [synth.covar_batch(feats)])[0].vals[0])
    th, it, ok = apps.ridge_bgd(C, len(feats), lam=1e-2, tol=1e-10)
    assert ok, it
    assert np.allclose(th, apps.ridge_closed_form(Cref, len(feats), 1e-2), rtol=1e-6, atol=1e-8)
    mdb = _mi_db(5, 30_000)
    attrs = ["a", "b", "c", "e"]
    b = synth.mi_batch(attrs)
    Mg = apps.mi_matrix(attrs, run_gpu(mdb, b))
    Mo = apps.mi_matrix(attrs, _results(mdb, b))
    assert np.allclose(Mg, Mo, rtol=1e-12, atol=1e-15)
    assert apps.chow_liu_tree(Mg) == apps.chow_liu_tree(Mo)


def _cart_numpy(J, features, target, thresholds, max_depth, min_split, categoricals=()):
    """The same CART over the materialised join (numpy masks)."""
    y = J[target].to_numpy()
    cols = {a: J[a].to_numpy().astype(np.float64) for a in list(features) + list(categoricals)}

    def node(mask, depth):
        n = mask.sum()
        s, s2 = y[mask].sum(), (y[mask] ** 2).sum()
        out = {"n": int(n), "mean": s / n if n else 0.0}
        if depth == max_depth or n < min_split:
            return out
        sse = s2 - s * s / n
        best = None

        def consider(lm, split):
            nonlocal best
            nl = lm.sum()
            nr = n - nl
            if nl == 0 or nr == 0:
                return
            sl, s2l = y[lm].sum(), (y[lm] ** 2).sum()
            sr, s2r = s - sl, s2 - s2l
            gain = sse - (s2l - sl * sl / nl) - (s2r - sr * sr / nr)
            if best is None or gain > best[0]:
                best = (gain, split)

        for a in features:
            for t in thresholds:
                consider(mask & (cols[a] <= t), ("num", a, t))
        for x in categoricals:
            vals = np.unique(cols[x][mask])
            cats = sorted(((y[mask & (cols[x] == c)].mean(), int(c)) for c in vals))
            for i in range(len(cats) - 1):
                left = [c for _, c in cats[:i + 1]]
                consider(mask & np.isin(cols[x], left), ("cat", x, left))
        if best is None or best[0] <= 0:
            return out
        split = best[1]
        if split[0] == "num":
            _, a, t = split
            out.update(feature=a, threshold=t, left=node(mask & (cols[a] <= t), depth + 1),
                       right=node(mask & (cols[a] > t), depth + 1))
        else:
            _, x, left = split
            lm = np.isin(cols[x], left)
            out.update(feature=x, categories=float(sum(1 << c for c in left)), left=node(mask & lm, depth + 1),
                       right=node(mask & ~lm, depth + 1))
        return out

    return node(np.ones(len(J), bool), 0)


def _same_tree(g, r):
    assert g["n"] == r["n"] and math.isclose(g["mean"], r["mean"], rel_tol=1e-9, abs_tol=1e-12)
    assert ("feature" in g) == ("feature" in r), (g.get("feature"), r.get("feature"))
    if "feature" in g:
        assert g["feature"] == r["feature"] and g.get("threshold") == r.get("threshold")
        assert g.get("categories") == r.get("categories")
        _same_tree(g["left"], r["left"])
        _same_tree(g["right"], r["right"])


@pytest.mark.gpu
@pytest.mark.parametrize("dynamic", [True, False])
def test_regression_tree_matches_numpy_cart(dynamic):
    """dynamic=True: one plan, the node's path condition rebound per node (lmfao_set_condition,
    PAPER.md P:2086-2092); dynamic=False: one plan per node."""
    from paper_1906_08687_b200 import lmfao
    w = synth.config3(seed=2, fact_rows=30_000, dim_rows=(40, 300, 2000))
    feats = ["x1", "x2", "x5", "d1_1", "d2_3", "d3_2"]
    ts = synth.thresholds_c3()
    e = lmfao.Engine()
    try:
        lmfao.load(e, w.db, [])
        tree = apps.regression_tree(e, feats, "y", ts, max_depth=3, min_split=2_000, dynamic=dynamic)
    finally:
        e.close()
    ref = _cart_numpy(_join(w.db), feats, "y", ts, 3, 2_000)
    _same_tree(tree, ref)
    assert "feature" in tree and "feature" in tree["left"]  # a non-trivial tree


def test_assign_roots_follows_the_weights():
    schemas = {"F": {"k1", "k2", "x"}, "D1": {"k1", "a", "b"}, "D2": {"k2", "c"}}
    sizes = {"F": 1000, "D1": 10, "D2": 20}
    Q = synth.Query
    batch = [Q(["a", "b"], []), Q(["a"], []), Q(["c"], []), Q([], []), Q(["k1"], []), Q(["x", "c"], [])]
    # weights: D1 1+1+1/3+1 (k1 is in F and D1) = 3.33, F 1/3+1+1/2 = 1.83, D2 1+1/3+1/2 = 1.83;
    # order D1, F (larger than D2), D2
    roots = apps.assign_roots(schemas, sizes, batch)
    assert roots == ["D1", "D1", "D2", "D1", "D1", "F"]  # F beats D2 on size for the tie
    # ties break towards the larger relation
    assert apps.assign_roots({"A": {"u"}, "B": {"u"}}, {"A": 5, "B": 9}, [Q([], [])]) == ["B"]


def test_reroot_keeps_the_tree():
    edges = [("F", "D1"), ("F", "D2"), ("D2", "E")]
    e = apps.reroot(edges, "E")
    assert set(map(frozenset, e)) == set(map(frozenset, edges))
    assert e[0] == ("E", "D2") and len(e) == 3


@pytest.mark.gpu
def test_batch_over_assigned_roots_matches_oracle():
    """Results do not depend on the root (reading R16): run each query at the root the
    heuristic assigns and compare with the oracle at the original root."""
    from _parity import assert_parity, run_gpu
    db = synth.random_db(21, max_rels=4, max_rows=600, unique_child_keys=True)
    batch = synth.random_batch(5, db, n_queries=5, groupby_ok=lambda a: True)
    schemas = {r.name: set(r.cols) for r in db.relations}
    sizes = {r.name: len(next(iter(r.cols.values()))) for r in db.relations}
    roots = apps.assign_roots(schemas, sizes, batch)
    ref = oracle.evaluate(db, batch)
    ran = 0
    for r in set(roots):
        sub = [q for q, rr in zip(batch, roots) if rr == r]
        rdb = synth.Database(db.relations, r, apps.reroot(db.edges, r))
        try:
            got = run_gpu(rdb, sub)
        except Exception as e:  # a shape the engine does not place at this root (e.g. deep group-bys)
            if "UNSUPPORTED" in str(e):
                continue
            raise
        assert_parity(got, [x for x, rr in zip(ref, roots) if rr == r], sub)
        ran += 1
    assert ran >= 1, roots


@pytest.mark.gpu
@pytest.mark.parametrize("dynamic", [True, False])
def test_regression_tree_with_categorical_splits(dynamic):
    """Categorical features split by set inclusion: node paths carry LMFAO_F_IN."""
    from paper_1906_08687_b200 import lmfao
    w = synth.config3(seed=3, fact_rows=30_000, dim_rows=(40, 300, 2000))
    rng = np.random.default_rng(9)
    F = w.db.rel("F")
    cat = rng.integers(0, 7, F.nrows).astype(np.int32)
    F.cols["cat"] = cat
    F.cols["y"] = F.cols["y"] + np.array([0.0, 3.0, -2.0, 1.0, 5.0, -4.0, 0.5])[cat]  # y depends on cat
    D = w.db.rel("D1")
    D.cols["dc"] = rng.integers(0, 5, D.nrows).astype(np.int32)
    feats = ["x1", "d2_3"]
    ts = synth.thresholds_c3()[::4]
    e = lmfao.Engine()
    try:
        lmfao.load(e, w.db, [])
        tree = apps.regression_tree(e, feats, "y", ts, max_depth=3, min_split=1_000, categoricals=["cat", "dc"],
                                    dynamic=dynamic)
    finally:
        e.close()
    ref = _cart_numpy(_join(w.db), feats, "y", ts, 3, 1_000, categoricals=["cat", "dc"])
    _same_tree(tree, ref)
    assert tree.get("feature") == "cat" and "categories" in tree
