"""Pins for the oracle (oracle/oracle.cpp) against things other than itself.

Every check here is independent of the oracle's code: literal hand-enumerated
values (tests/golden/*.json, each with its citation), a brute-force pandas
materialisation of the join, closed forms computed from key frequencies, numpy
library routines on special cases, and the paper's worked decompositions
(Ex. 4.1/4.2, the §4.3 chain) computed view by view.  A dropped term, a wrong
sign or index, a transposed operand or a wrong join semantics in the oracle
fails at least one of them.
"""
import itertools
import json
import math
import os

import numpy as np
import pandas as pd
import pytest

import oracle
import synth
from synth import F_CONST, F_EQ, F_GE, F_GT, F_IDENT, F_LE, F_LT, F_NE, Factor, Product, Query

from _udaf import parse_udaf, query

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _db(name):
    return {"h1": synth.hand_h1, "h2": synth.hand_h2, "h3": synth.hand_h3, "h4": synth.hand_h4,
            "h5": lambda: synth.hand_h2(root="S")}[name]()


@pytest.mark.parametrize("name", ["h1", "h2", "h3", "h4", "h5"])
def test_hand_databases(name):
    g = json.load(open(os.path.join(GOLD, f"{name}.json")))
    qs = g["queries"]
    if qs == "same-as-h2":
        qs = json.load(open(os.path.join(GOLD, "h2.json")))["queries"]
    db = _db(name)
    batch = [query(q["groupby"], q["udafs"]) for q in qs]
    res = oracle.evaluate(db, batch)
    for q, r in zip(qs, res):
        assert r.keys.tolist() == q["keys"] or (len(q["keys"]) == 0 and r.keys.shape[0] == 0)
        assert r.counts.tolist() == q["counts"]
        exp = np.array(q["vals"], dtype=np.float64).reshape(r.vals.shape)
        assert np.array_equal(r.vals, exp), (name, q, r.vals)


def test_chain_closed_form_left_right_views():
    """§4.3: Q_i(X_i; c1*c2) += L_i(X_i; c1), R_i(X_i; c2), with
    L_i over S_i..S_{n-1} (right to left) and R_i over S_1..S_{i-1}."""
    db = synth.hand_h3()
    S = [list(zip(db.rel(f"S{i}").cols[f"X{i}"].tolist(), db.rel(f"S{i}").cols[f"X{i+1}"].tolist())) for i in (1, 2, 3)]
    n = 4
    dom = [sorted({t[0] for t in S[0]})] + [sorted({t[1] for t in S[i]}) for i in range(3)]
    L = {n: {v: 1 for v in dom[n - 1]}}
    for i in range(n - 1, 0, -1):
        L[i] = {}
        for a, b in S[i - 1]:
            L[i][a] = L[i].get(a, 0) + L[i + 1].get(b, 0)
    R = {1: {v: 1 for v in dom[0]}}
    for i in range(2, n + 1):
        R[i] = {}
        for a, b in S[i - 2]:
            R[i][b] = R[i].get(b, 0) + R[i - 1].get(a, 0)
    batch = [query([f"X{i}"], ["1"]) for i in range(1, n + 1)]
    res = oracle.evaluate(db, batch)
    for i, r in zip(range(1, n + 1), res):
        expect = {v: L[i].get(v, 0) * R[i].get(v, 0) for v in set(L[i]) | set(R[i])}
        expect = {k: v for k, v in expect.items() if v}
        got = {int(k[0]): int(c) for k, c in zip(r.keys, r.vals[:, 0])}
        assert got == expect


def _materialise(db):
    """Independent brute force: pandas natural join along the tree edges."""
    frames = {r.name: pd.DataFrame({c: v for c, v in r.cols.items()}) for r in db.relations}
    order = [db.root]
    children = {}
    for p, c in db.edges:
        children.setdefault(p, []).append(c)
    i = 0
    while i < len(order):
        order += children.get(order[i], [])
        i += 1
    J = frames[db.root]
    for name in order[1:]:
        f = frames[name]
        on = [c for c in f.columns if c in J.columns]
        J = J.merge(f, on=on, how="inner")
    return J


def _eval_products(J, udaf):
    tot = np.zeros(len(J))
    for p in udaf:
        v = np.full(len(J), p.coeff)
        for f in p.factors:
            if f.kind == F_CONST:
                x = np.full(len(J), f.param)
            else:
                a = J[f.attr].to_numpy().astype(np.float64)
                if f.kind == synth.F_IN:  # set inclusion: the members of the mask, written out
                    members = [v for v in range(53) if (int(f.param) >> v) & 1]
                    x = np.isin(a, np.array(members, dtype=np.float64)) * 1.0
                else:
                    x = {F_IDENT: a, F_LT: (a < f.param) * 1.0, F_LE: (a <= f.param) * 1.0, F_GT: (a > f.param) * 1.0,
                         F_GE: (a >= f.param) * 1.0, F_EQ: (a == f.param) * 1.0, F_NE: (a != f.param) * 1.0}[f.kind]
            v = v * x
        tot = tot + v
    return tot


def _brute(db, batch):
    J = _materialise(db)
    out = []
    for q in batch:
        vals = np.stack([_eval_products(J, u) for u in q.udafs], axis=1) if q.udafs else np.zeros((len(J), 0))
        if not q.groupby:
            out.append((np.zeros((1, 0), np.int64), vals.sum(axis=0, keepdims=True), np.array([len(J)])))
            continue
        if len(J) == 0:
            out.append((np.zeros((0, len(q.groupby)), np.int64), np.zeros((0, len(q.udafs))), np.zeros(0)))
            continue
        df = J[q.groupby].copy()
        for j in range(vals.shape[1]):
            df[f"_u{j}"] = vals[:, j]
        df["_n"] = 1
        g = df.groupby(q.groupby, sort=True).sum()
        keys = np.array(list(g.index), dtype=np.int64).reshape(len(g), len(q.groupby))
        out.append((keys, g[[f"_u{j}" for j in range(vals.shape[1])]].to_numpy(), g["_n"].to_numpy()))
    return out


@pytest.mark.parametrize("seed", range(40))
def test_random_acyclic_dbs_vs_pandas_materialisation(seed):
    """S:636 style: oracle == brute-force materialisation on random acyclic DBs
    (<=5 relations, <=1000 rows, key domains <=50)."""
    db = synth.random_db(seed, max_rows=60 if seed % 2 else 400)
    batch = synth.random_batch(seed, db, n_queries=4)
    res = oracle.evaluate(db, batch)
    ref = _brute(db, batch)
    for r, (k, v, n) in zip(res, ref):
        assert r.keys.tolist() == k.tolist()
        assert r.counts.tolist() == [int(x) for x in n]
        # dyadic inputs: sums are exact or within a few ulps of reassociation
        assert np.allclose(r.vals, v, rtol=1e-12, atol=1e-9), (r.vals, v)


def _count_closed_form(db):
    """COUNT of a star join from key frequencies (never enumerates):
    Σ_f Π_r mult_r(k_r(f)) (SURVEY §8(c) closed forms)."""
    F = db.rel(db.root)
    w = np.ones(F.nrows, dtype=np.int64)
    for p, c in db.edges:
        assert p == db.root
        C = db.rel(c)
        key = [k for k in C.cols if k in F.cols][0]
        vals, cnt = np.unique(C.cols[key], return_counts=True)
        idx = np.searchsorted(vals, F.cols[key])
        idx = np.minimum(idx, len(vals) - 1)
        m = np.where(vals[idx] == F.cols[key], cnt[idx], 0)
        w *= m
    return int(w.sum())


@pytest.mark.parametrize("cfg", ["C1", "C2", "C4"])
def test_count_equals_key_frequency_closed_form(cfg):
    w = {"C1": lambda: synth.config1(), "C2": lambda: synth.config2(fact_rows=30_000, dim_rows=(50, 300, 2000)),
         "C4": lambda: synth.config4(fact_rows=30_000, dim_rows=(50, 300, 2000))}[cfg]()
    r = oracle.evaluate(w.db, [query([], ["1"])])[0]
    cf = _count_closed_form(w.db)
    assert int(r.counts[0]) == cf == int(r.vals[0, 0])
    # no dangling keys in the configs (reading R7): COUNT = fact rows
    assert cf == w.db.rel("F").nrows


def test_duplicate_keys_multiply_closed_form():
    db = synth.random_db(7, star=True, max_rows=300)
    r = oracle.evaluate(db, [query([], ["1"])])[0]
    assert int(r.counts[0]) == _count_closed_form(db)


def test_single_relation_covariance_is_xtx_fsum():
    rng = np.random.default_rng(3)
    X = rng.standard_normal((500, 4))
    R = synth.Relation("R", {f"x{i}": X[:, i].copy() for i in range(4)})
    db = synth.Database([R], "R", [])
    q = synth.covar_batch([f"x{i}" for i in range(4)])
    r = oracle.evaluate(db, [q])[0]
    Z = np.concatenate([np.ones((500, 1)), X], axis=1)
    exp = [math.fsum(Z[:, 0] * Z[:, 0])] + [math.fsum(Z[:, 0] * Z[:, i + 1]) for i in range(4)]
    for i in range(4):
        for j in range(i, 4):
            exp.append(math.fsum(X[:, i] * X[:, j]))
    assert np.allclose(r.vals[0], exp, rtol=1e-15, atol=0)


def test_config1_matches_numpy_fancy_index_materialisation():
    w = synth.config1()
    F, S, T = (w.db.rel(n) for n in "FST")
    si = {int(k): i for i, k in enumerate(S.cols["a"])}
    ti = {int(k): i for i, k in enumerate(T.cols["b"])}
    ia = np.array([si[int(k)] for k in F.cols["a"]])
    ib = np.array([ti[int(k)] for k in F.cols["b"]])
    cols = {"x1": F.cols["x1"], "x2": F.cols["x2"], "x3": F.cols["x3"], "x4": S.cols["x4"][ia],
            "x5": S.cols["x5"][ia], "x6": T.cols["x6"][ib]}
    r = oracle.evaluate(w.db, w.batch)[0]
    feats = w.meta["features"]
    exp = [float(F.nrows)] + [math.fsum(cols[a]) for a in feats]
    for i, a in enumerate(feats):
        for b in feats[i:]:
            exp.append(math.fsum(cols[a] * cols[b]))
    assert r.vals.shape == (1, 28)
    assert np.allclose(r.vals[0], exp, rtol=1e-13)


def test_covariance_symmetric_and_psd():
    w = synth.config2(fact_rows=20_000, dim_rows=(40, 200, 1000))
    feats = w.meta["features"][:6] + w.meta["features"][8:10] + w.meta["features"][-3:]
    n = len(feats)
    udafs = ["1"] + feats + [f"{a}*{b}" for a in feats for b in feats]
    r = oracle.evaluate(w.db, [query([], udafs)])[0].vals[0]
    M = np.zeros((n + 1, n + 1))
    M[0, 0] = r[0]
    M[0, 1:] = M[1:, 0] = r[1:n + 1]
    M[1:, 1:] = r[n + 1:].reshape(n, n)
    assert np.array_equal(M, M.T)  # x*y and y*x enumerate the same tuples
    np.linalg.cholesky(M + 1e-9 * np.eye(n + 1))


def test_contingency_marginals_exact():
    """Σ_b C_ij[a,b] = C_i[a] and Σ_a C_i[a] = COUNT, bit-exact."""
    w = synth.config4(fact_rows=20_000, dim_rows=(50, 300, 2000))
    names = w.meta["attrs"]
    sub = [names[0], names[1], names[5], names[10]]  # spans F, D1, D2(?) and D3 homes
    batch = synth.mi_batch(sub)
    res = oracle.evaluate(w.db, batch)
    pairs = list(itertools.combinations(sub, 2))
    single = {a: res[len(pairs) + i] for i, a in enumerate(sub)}
    total = int(res[-1].counts[0])
    for (a, b), r in zip(pairs, res):
        for pos, att in ((0, a), (1, b)):
            marg = {}
            for k, c in zip(r.keys[:, pos], r.counts):
                marg[int(k)] = marg.get(int(k), 0) + int(c)
            s = single[att]
            assert marg == {int(k[0]): int(c) for k, c in zip(s.keys, s.counts)}
            assert np.array_equal(r.vals[:, 0], r.counts.astype(np.float64))
    for a in sub:
        assert int(single[a].counts.sum()) == total


def test_cube_rollups():
    """Each coarser cuboid cell = Σ of its finer cells (counts exact, sums 1e-12)."""
    w = synth.config5(fact_rows=20_000, dim_rows=(40, 300, 2000, 5000), cube_doms=(5, 20, 50))
    cube = w.batch[:8]
    res = oracle.evaluate(w.db, cube)
    by = {tuple(q.groupby): r for q, r in zip(cube, res)}
    full = by[("A", "B", "C")]
    for gb, r in by.items():
        pos = [("A", "B", "C").index(a) for a in gb]
        agg = {}
        for k, v, c in zip(full.keys, full.vals, full.counts):
            kk = tuple(int(k[p]) for p in pos)
            a = agg.setdefault(kk, [np.zeros(5), 0])
            a[0] = a[0] + v
            a[1] += int(c)
        assert sorted(agg) == [tuple(int(x) for x in k) for k in r.keys]
        for k, v, c in zip(r.keys, r.vals, r.counts):
            a = agg[tuple(int(x) for x in k)]
            assert a[1] == int(c)
            assert np.allclose(v, a[0], rtol=1e-12)


def test_regression_tree_batch_properties():
    w = synth.config3(fact_rows=20_000, dim_rows=(40, 300, 2000))
    res = oracle.evaluate(w.db, w.batch)
    pred = res[-1].vals[0]
    base = pred[:3]
    assert base[0] == w.db.rel("F").nrows
    per = pred[3:].reshape(len(w.meta["features"]), 20, 3)
    assert np.all(np.diff(per[:, :, 0], axis=1) >= 0)  # counts non-decreasing in t
    assert np.all(per[:, :, 0] <= base[0])
    for i, r in enumerate(res[:-1]):  # Σ over categories = unconditioned totals
        assert int(r.counts.sum()) == int(base[0])
        assert np.allclose(r.vals.sum(axis=0), base, rtol=1e-12)
        n, s, s2 = r.vals.T
        assert np.all(s2 / n - (s / n) ** 2 >= -1e-12)  # variance >= 0


def _favorita_toy(seed=5):
    """A toy Favorita-shaped DB (Fig. 2 schema): S(date,store,item,units),
    T(date,store,txns), R(store,city), O(date,price), H(date,htype), I(item,family)."""
    rng = np.random.default_rng(seed)
    nd, ns, ni = 6, 4, 5
    i32 = lambda a: np.asarray(a, np.int32)
    d = lambda a: np.round(np.asarray(a, np.float64) * 8) / 8
    S = synth.Relation("S", {"date": i32(rng.integers(0, nd, 80)), "store": i32(rng.integers(0, ns, 80)),
                             "item": i32(rng.integers(0, ni, 80)), "units": d(rng.uniform(0, 4, 80))})
    T = synth.Relation("T", {"date": i32(rng.integers(0, nd, 30)), "store": i32(rng.integers(0, ns, 30)),
                             "txns": d(rng.uniform(0, 9, 30))})
    R = synth.Relation("R", {"store": i32(rng.integers(0, ns, 6)), "city": i32(rng.integers(0, 3, 6))})
    O = synth.Relation("O", {"date": i32(rng.integers(0, nd, 9)), "price": d(rng.uniform(1, 3, 9))})
    H = synth.Relation("H", {"date": i32(rng.integers(0, nd, 7)), "htype": i32(rng.integers(0, 2, 7))})
    I = synth.Relation("I", {"item": i32(rng.integers(0, ni, 8)), "family": i32(rng.integers(0, 3, 8))})
    db = synth.Database([S, T, R, O, H, I], "S", [("S", "T"), ("T", "R"), ("T", "O"), ("S", "H"), ("S", "I")])
    return db


def _groupsum(keys, vals):
    out = {}
    for k, v in zip(keys, vals):
        out[k] = out.get(k, 0.0) + v
    return out


def test_paper_example_4_1_and_4_2_view_decomposition():
    """Ex. 4.1: Q1(units*price) via V_O, V_R, V_T, V_H, V_I; Ex. 4.2
    (P:754-765): Q2(family; price) via V'_I(family,item;1)."""
    db = _favorita_toy()
    S, T, R, O, H, I = (db.rel(n) for n in "STROHI")
    V_O = _groupsum(O.cols["date"].tolist(), O.cols["price"].tolist())
    V_R = _groupsum(R.cols["store"].tolist(), [1.0] * R.nrows)
    V_T = {}
    for dd, ss in zip(T.cols["date"].tolist(), T.cols["store"].tolist()):
        V_T[(dd, ss)] = V_T.get((dd, ss), 0.0) + V_R.get(ss, 0.0) * V_O.get(dd, 0.0)
    V_H = _groupsum(H.cols["date"].tolist(), [1.0] * H.nrows)
    V_I = _groupsum(I.cols["item"].tolist(), [1.0] * I.nrows)
    Q1 = 0.0
    for dd, ss, it, u in zip(S.cols["date"].tolist(), S.cols["store"].tolist(), S.cols["item"].tolist(),
                             S.cols["units"].tolist()):
        Q1 += u * V_T.get((dd, ss), 0.0) * V_H.get(dd, 0.0) * V_I.get(it, 0.0)
    V_Ip = _groupsum(list(zip(I.cols["family"].tolist(), I.cols["item"].tolist())), [1.0] * I.nrows)
    Q2 = {}
    for dd, ss, it in zip(S.cols["date"].tolist(), S.cols["store"].tolist(), S.cols["item"].tolist()):
        for (fam, item), c2 in V_Ip.items():
            if item == it:
                v = V_T.get((dd, ss), 0.0) * c2 * V_H.get(dd, 0.0)
                if V_T.get((dd, ss), 0.0) and V_H.get(dd, 0.0):
                    Q2[fam] = Q2.get(fam, 0.0) + v
    res = oracle.evaluate(db, [query([], ["units*price"]), query(["family"], ["price"])])
    assert res[0].vals[0, 0] == pytest.approx(Q1, rel=1e-14)
    got = {int(k[0]): v for k, v in zip(res[1].keys, res[1].vals[:, 0])}
    assert sorted(got) == sorted(Q2)
    for k in Q2:
        assert got[k] == pytest.approx(Q2[k], rel=1e-14)


def test_factor_kinds_semantics():
    """Each Kronecker op on H1's join (x ∈ {2,2,3,3,5}): P:345 '1 if the
    condition is true and 0 otherwise'."""
    ops = {"[x<3]": 2, "[x<=3]": 4, "[x>3]": 1, "[x>=3]": 3, "[x==3]": 2, "[x!=3]": 3, "2.5": 12.5,
           "-1*x": -15, "x+[x>=5]*10": 25, "0.5*x*x": 25.5}
    r = oracle.evaluate(synth.hand_h1(), [query([], list(ops))])[0]
    assert r.vals[0].tolist() == list(map(float, ops.values()))


def test_batch_size_formulas():
    g = json.load(open(os.path.join(GOLD, "batch_sizes.json")))
    assert synth.n_aggregates(synth.config1(fact_rows=10).batch) == g["C1"] == (6 + 1) * (6 + 2) // 2
    c2 = synth.covar_batch([f"f{i}" for i in range(38)])
    assert len(c2.udafs) == g["C2"] == 39 * 40 // 2
    rt = synth.rt_batch([f"f{i}" for i in range(38)], "y", ["c"], synth.thresholds_c3())
    assert len(rt[-1].udafs) - 3 == g["C3_predicate_aggregates"] == 1 * 38 * 3 * 20
    mi = synth.mi_batch([f"a{i}" for i in range(12)])
    assert sum(1 for q in mi if len(q.groupby) == 2) == g["C4_pairs"] == 12 * 11 // 2
    assert sum(1 for q in mi if len(q.groupby) == 1) == g["C4_singles"]
    cube = synth.cube_batch(["A", "B", "C"], [f"m{i}" for i in range(5)])
    assert synth.n_aggregates(cube) == g["C5_cube"] == 2 ** 3 * 5
    assert synth.C4_DOMS == [2, 4, 6, 11, 19, 34, 59, 104, 184, 323, 568, 1000]


def test_root_range_shards_sum_to_whole():
    """Row-sharding the root is exact for counts and linear for sums."""
    w = synth.config2(fact_rows=9_000, dim_rows=(30, 100, 400))
    b = [query([], ["1", "x1", "x1*d3_1", "d1_2*d2_3"])]
    full = oracle.evaluate(w.db, b)[0]
    parts = [oracle.evaluate(w.db, b, root_range=(lo, lo + 3000))[0] for lo in (0, 3000, 6000)]
    assert sum(int(p.counts[0]) for p in parts) == int(full.counts[0])
    assert np.allclose(sum(p.vals[0] for p in parts), full.vals[0], rtol=1e-13)


def test_errors():
    db = synth.hand_h1()
    with pytest.raises(ValueError, match="unknown attribute"):
        oracle.evaluate(db, [query([], ["zz"])])
    with pytest.raises(ValueError, match="group-by attribute must be int"):
        oracle.evaluate(db, [query(["x"], ["1"])])
    bad = synth.Database(db.relations, "F", [("F", "S"), ("S", "F")])
    with pytest.raises(ValueError):
        oracle.evaluate(bad, [query([], ["1"])])
    # running intersection violated: R(A,B)-S(B,C)-T(A,C) as a path
    i = lambda v: np.asarray(v, np.int32)
    Rr = synth.Relation("R", {"A": i([1]), "B": i([1])})
    Ss = synth.Relation("S", {"B": i([1]), "C": i([1])})
    Tt = synth.Relation("T", {"A": i([1]), "C": i([1])})
    with pytest.raises(ValueError, match="running intersection"):
        oracle.evaluate(synth.Database([Rr, Ss, Tt], "R", [("R", "S"), ("S", "T")]), [query([], ["1"])])


@pytest.mark.parametrize("seed", range(8))
def test_set_inclusion_factor_vs_pandas(seed):
    """LMFAO_F_IN (reading R20): 1[x ∈ S] for a bit mask S over {0..52}, against membership in
    the listed set on the materialised join; values outside [0, 52], negative and fractional
    values are never members."""
    db = synth.random_db(100 + seed, max_rows=300)
    rng = np.random.default_rng(seed)
    attrs = [(r.name, c) for r in db.relations for c in r.cols]
    batch = []
    for _ in range(3):
        name, col = attrs[rng.integers(len(attrs))]
        mask = float(int(rng.integers(0, 2 ** 20)) | (1 << 52) | 1)
        other = attrs[rng.integers(len(attrs))][1]
        batch.append(synth.Query([], [[synth.Product(1.0, (synth.Factor(synth.F_IN, col, mask),))],
                                     [synth.Product(2.0, (synth.Factor(synth.F_IN, col, mask), synth.ident(other)))]]))
    res = oracle.evaluate(db, batch)
    ref = _brute(db, batch)
    for r, (k, v, n) in zip(res, ref):
        assert np.allclose(r.vals, v, rtol=1e-12, atol=1e-9), (r.vals, v)


@pytest.mark.parametrize("name", ["h1", "h2", "h3", "h4", "h5"])
@pytest.mark.parametrize("threads,acc", [(3, "longdouble"), (1, "neumaier"), (4, "neumaier")])
def test_hand_databases_threads_and_neumaier(name, threads, acc):
    """The OpenMP fact-row chunks (private tables merged in chunk order) and the Neumaier
    accumulation mode reproduce the literal hand values
    (all dyadic: every mode must be exact)."""
    g = json.load(open(os.path.join(GOLD, f"{name}.json")))
    qs = g["queries"]
    if qs == "same-as-h2":
        qs = json.load(open(os.path.join(GOLD, "h2.json")))["queries"]
    batch = [query(q["groupby"], q["udafs"]) for q in qs]
    res = oracle.evaluate(_db(name), batch, threads=threads, acc=acc)
    for q, r in zip(qs, res):
        assert r.keys.tolist() == q["keys"] or (len(q["keys"]) == 0 and r.keys.shape[0] == 0)
        assert r.counts.tolist() == q["counts"]
        assert np.array_equal(r.vals, np.array(q["vals"], dtype=np.float64).reshape(r.vals.shape))


@pytest.mark.parametrize("seed", range(6))
def test_threads_vs_pandas_materialisation(seed):
    """Chunked enumeration (including chunks with no joined tuple and more threads than
    root rows) against the brute-force pandas materialisation."""
    db = synth.random_db(200 + seed, max_rows=40 if seed % 2 else 300)
    batch = synth.random_batch(seed, db, n_queries=3)
    ref = _brute(db, batch)
    for t in (2, 7, 64):
        for r, (k, v, n) in zip(oracle.evaluate(db, batch, threads=t), ref):
            assert r.keys.tolist() == k.tolist()
            assert r.counts.tolist() == [int(x) for x in n]
            assert np.allclose(r.vals, v, rtol=1e-12, atol=1e-9)


def test_oracle_self_bound_longdouble_vs_neumaier():
    """SURVEY.md §8(c) "GPU acceptance": the oracle's own rounding error, bounded by running
    it in its two accumulation modes (long double vs Neumaier-compensated double) on a
    covariance and a cube batch: |ld - neumaier| <= 1e-13·A (A = Σ|term|) everywhere, far
    inside the 1e-9 / 1e-12·A acceptance band the GPU is held to (reading R14)."""
    w = synth.config5(fact_rows=60_000, dim_rows=(50, 300, 2_000, 10_000))
    a = oracle.evaluate(w.db, w.batch, threads=0)
    b = oracle.evaluate(w.db, w.batch, threads=0, acc="neumaier")
    worst = 0.0
    for ra, rb in zip(a, b):
        assert np.array_equal(ra.keys, rb.keys) and np.array_equal(ra.counts, rb.counts)
        d = np.abs(ra.vals - rb.vals)
        assert (d <= 1e-13 * ra.absmass).all()
        worst = max(worst, float(np.max(d / np.maximum(ra.absmass, 1e-300))))
    assert worst < 1e-13
