"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method: it only draws relations (columns
of int32 keys/categoricals and float64 features) and spells out aggregate batches
as plain data (queries -> UDAFs -> products -> factors).
Both `oracle/` and `paper_1906_08687_b200/` consume these objects through their
own, separate marshalling code.

Workload recipes follow BASELINE.json `configs` and the readings in SURVEY.md
§8(c) (listed again in DESIGN.md §3 "Readings"):
  * dimension primary keys: seeded distinct non-negative int32 values in random
    row order (reading R7);
  * foreign keys: finite Zipf(s) over the dimension's keys, rank -> key through a
    seeded permutation (reading R6);
  * categorical values: Zipf rank i -> value i-1 (C4) or uniform (C3, C5);
  * C3 thresholds t_i = (2i-21)/8, i = 1..20, predicate x <= t (reading R5).
The paper's datasets (Retailer, Favorita, Yelp, TPC-DS) are not available; these
synthetic snowflakes stand in for them ("large fact table in the
center and several smaller dimension tables").
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np

# factor kinds (constant, identity, Kronecker 1_{X op t})
F_CONST, F_IDENT, F_LT, F_LE, F_GT, F_GE, F_EQ, F_NE, F_IN = range(9)


@dataclass
class Relation:
    name: str
    cols: dict  # name -> np.ndarray (int32 or float64), all the same length

    @property
    def nrows(self) -> int:
        return len(next(iter(self.cols.values()))) if self.cols else 0


@dataclass
class Database:
    relations: list
    root: str
    edges: list  # (parent, child) relation names

    def rel(self, name: str) -> Relation:
        for r in self.relations:
            if r.name == name:
                return r
        raise KeyError(name)


@dataclass(frozen=True)
class Factor:
    kind: int
    attr: str | None = None
    param: float = 0.0


@dataclass(frozen=True)
class Product:
    coeff: float
    factors: tuple = ()


@dataclass
class Query:
    groupby: list
    udafs: list  # list of list[Product]
    name: str = ""


@dataclass
class Workload:
    name: str
    db: Database
    batch: list  # list[Query]
    meta: dict = field(default_factory=dict)


# ----------------------------------------------------------------------------- RNG
def _rng(seed: int, *path) -> np.random.Generator:
    """Independent stream per (seed, relation, column) (reading R13)."""
    words = [int(seed) & 0xFFFFFFFF]
    for p in path:
        if isinstance(p, str):
            words.extend(p.encode())
        else:
            words.append(int(p) & 0xFFFFFFFF)
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(words)))


def distinct_keys(rng: np.random.Generator, n: int) -> np.ndarray:
    """n distinct non-negative int32 values in random order (reading R7)."""
    out = np.empty(0, dtype=np.int64)
    while out.size < n:
        cand = rng.integers(0, 2**31 - 1, size=int(n * 1.2) + 16, dtype=np.int64)
        out = np.unique(np.concatenate([out, cand]))
    out = rng.permutation(out)[:n]
    return out.astype(np.int32)


def zipf_ranks(rng: np.random.Generator, n_values: int, s: float, size: int) -> np.ndarray:
    """Finite Zipf: P(rank i) ∝ i^-s, i = 1..n_values, by inverse CDF (reading R6).
    Returns 0-based ranks."""
    w = np.arange(1, n_values + 1, dtype=np.float64) ** (-s)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    u = rng.random(size)
    r = np.searchsorted(cdf, u, side="right")
    return np.minimum(r, n_values - 1).astype(np.int64)


def zipf_fk(seed: int, rel: str, col: str, dim_keys: np.ndarray, s: float, size: int) -> np.ndarray:
    rng = _rng(seed, rel, col)
    perm = rng.permutation(dim_keys.size)
    return dim_keys[perm[zipf_ranks(rng, dim_keys.size, s, size)]].astype(np.int32)


def uniform_fk(seed: int, rel: str, col: str, dim_keys: np.ndarray, size: int) -> np.ndarray:
    rng = _rng(seed, rel, col)
    return dim_keys[rng.integers(0, dim_keys.size, size)].astype(np.int32)


def normal(seed, rel, col, size):
    return _rng(seed, rel, col).standard_normal(size)


def uniform01(seed, rel, col, size):
    return _rng(seed, rel, col).random(size)


# -------------------------------------------------------------------- batch builders
def ident(a):
    return Factor(F_IDENT, a)


def const(c):
    return Factor(F_CONST, None, float(c))


def covar_batch(features: list) -> Query:
    """Ridge-LR covariance batch: COUNT, SUM(x_i), SUM(x_i*x_j), i<=j.
    ½(n+1)(n+2) aggregates for n features."""
    udafs = [[Product(1.0, ())]]
    udafs += [[Product(1.0, (ident(a),))] for a in features]
    for i, a in enumerate(features):
        for b in features[i:]:
            udafs.append([Product(1.0, (ident(a), ident(b)))])
    return Query([], udafs, name="covar")


def thresholds_c3():
    """Reading R5: t_i = (2i-21)/8, i=1..20 (dyadic, exact in binary)."""
    return [(2 * i - 21) / 8.0 for i in range(1, 21)]


def rt_batch(features, target, categoricals, thresholds):
    """Regression-tree node batch: per categorical X: Q(X; Σ1, Σy, Σy²);
    per predicate x <= t: Σ[x<=t], Σ y[x<=t], Σ y²[x<=t]; plus the unconditioned triple."""
    y = ident(target)
    qs = []
    for c in categoricals:
        qs.append(Query([c], [[Product(1.0, ())], [Product(1.0, (y,))], [Product(1.0, (y, y))]], name=f"rt_cat_{c}"))
    udafs = [[Product(1.0, ())], [Product(1.0, (y,))], [Product(1.0, (y, y))]]
    for a in features:
        for t in thresholds:
            p = Factor(F_LE, a, float(t))
            udafs.append([Product(1.0, (p,))])
            udafs.append([Product(1.0, (y, p))])
            udafs.append([Product(1.0, (y, y, p))])
    qs.append(Query([], udafs, name="rt_pred"))
    return qs


def mi_batch(attrs):
    """Chow-Liu / MI count queries Q_S for S ⊆ {i,j}: all pairs, all
    singles, and COUNT (Q_∅)."""
    qs = [Query([a, b], [[Product(1.0, ())]], name=f"mi_{a}_{b}") for a, b in itertools.combinations(attrs, 2)]
    qs += [Query([a], [[Product(1.0, ())]], name=f"mi_{a}") for a in attrs]
    qs.append(Query([], [[Product(1.0, ())]], name="mi_count"))
    return qs


def cube_batch(dims, measures):
    """Data cube: one query per subset F_i ⊆ S_k, each with SUM(m) for
    every measure (2^k·v aggregates)."""
    qs = []
    for k in range(len(dims) + 1):
        for sub in itertools.combinations(dims, k):
            qs.append(Query(list(sub), [[Product(1.0, (ident(m),))] for m in measures], name="cube_" + "".join(sub)))
    return qs


def n_aggregates(batch) -> int:
    return sum(len(q.udafs) for q in batch)


# ----------------------------------------------------------------------- configs
def _scale_rows(n, scale):
    return max(1, int(round(n * scale)))


def config1(seed: int = 0, fact_rows: int = 20_000) -> Workload:
    """BJ configs[0]: tiny star F(a,b,x1..x3~U(0,1)) 20k; S(a,x4,x5~N(0,1)) 200;
    T(b,x6) 50 (x6 ~ N(0,1), reading R9); keys uniform; 28 aggregates."""
    S_keys = distinct_keys(_rng(seed, "S", "a"), 200)
    T_keys = distinct_keys(_rng(seed, "T", "b"), 50)
    n = fact_rows
    F = Relation("F", {
        "a": uniform_fk(seed, "F", "a", S_keys, n),
        "b": uniform_fk(seed, "F", "b", T_keys, n),
        "x1": uniform01(seed, "F", "x1", n),
        "x2": uniform01(seed, "F", "x2", n),
        "x3": uniform01(seed, "F", "x3", n),
    })
    S = Relation("S", {"a": S_keys, "x4": normal(seed, "S", "x4", 200), "x5": normal(seed, "S", "x5", 200)})
    T = Relation("T", {"b": T_keys, "x6": normal(seed, "T", "x6", 50)})
    db = Database([F, S, T], "F", [("F", "S"), ("F", "T")])
    feats = ["x1", "x2", "x3", "x4", "x5", "x6"]
    return Workload("C1", db, [covar_batch(feats)], {"fact_rows": n, "features": feats})


def _snowflake(seed, fact_rows, dim_rows, dim_feats, fact_feats, s=1.1, fact_feat_dist="normal", tag="C2"):
    """Star with one FK per dim (reading R8): dims D1..DR with PK k_r + features."""
    rels = []
    fact = {}
    dims = []
    for r, (nr, nf) in enumerate(zip(dim_rows, dim_feats), start=1):
        key = f"k{r}"
        keys = distinct_keys(_rng(seed, tag, f"D{r}", key), nr)
        cols = {key: keys}
        for j in range(1, nf + 1):
            cols[f"d{r}_{j}"] = normal(seed, f"D{r}", f"d{r}_{j}", nr)
        dims.append(Relation(f"D{r}", cols))
        fact[key] = zipf_fk(seed, "F", key, keys, s, fact_rows)
    for j, name in enumerate(fact_feats):
        if fact_feat_dist == "normal":
            fact[name] = normal(seed, "F", name, fact_rows)
        else:
            fact[name] = fact_feat_dist(seed, name, fact_rows)
    F = Relation("F", fact)
    rels = [F] + dims
    return Database(rels, "F", [("F", d.name) for d in dims])


C2_DIMS = (1_000, 10_000, 100_000)


def config2(seed: int = 0, fact_rows: int = 10_000_000, dim_rows=C2_DIMS) -> Workload:
    """BJ configs[1]: covariance batch, fact 10M x (3 FK Zipf 1.1 + 8 N(0,1)),
    dims 1k/10k/100k x 10 N(0,1) features; 780 aggregates over 38 features."""
    fact_feats = [f"x{j}" for j in range(1, 9)]
    db = _snowflake(seed, fact_rows, dim_rows, (10, 10, 10), fact_feats)
    feats = fact_feats + [f"d{r}_{j}" for r in (1, 2, 3) for j in range(1, 11)]
    return Workload("C2", db, [covar_batch(feats)], {"fact_rows": fact_rows, "features": feats})


def config3(seed: int = 0, fact_rows: int = 10_000_000, dim_rows=C2_DIMS) -> Workload:
    """BJ configs[2]: regression-tree split batch on the C2 snowflake + y ~ N(0,1)
    and 5 categoricals with domains 10, 56, 316, 1778, 10000 (reading R10)."""
    w = config2(seed, fact_rows, dim_rows)
    db = w.db
    F = db.rel("F")
    F.cols["y"] = normal(seed, "F", "y", fact_rows)
    doms = {"c1": 10, "c2": 56, "c3": 316, "c4": 1778, "c5": 10000}
    place = {"c1": "F", "c5": "F", "c2": "D1", "c3": "D2", "c4": "D3"}
    for c, d in doms.items():
        R = db.rel(place[c])
        R.cols[c] = _rng(seed, place[c], c).integers(0, d, R.nrows).astype(np.int32)
    feats = w.meta["features"]
    batch = rt_batch(feats, "y", list(doms), thresholds_c3())
    return Workload("C3", db, batch, {"fact_rows": fact_rows, "features": feats, "categoricals": doms})


C4_DOMS = [int(round(2 * 500 ** (i / 11))) for i in range(12)]


def config4(seed: int = 0, fact_rows: int = 30_000_000, dim_rows=C2_DIMS) -> Workload:
    """BJ configs[3]: Chow-Liu pairwise counts; 12 categoricals (domains
    round(2*500^(i/11)), Zipf 1.0 values) with attribute i in relation i mod 4
    (reading R11); fact 30M with 3 FK Zipf 1.1; batch 66 pairs + 12 singles + COUNT."""
    db = _snowflake(seed, fact_rows, dim_rows, (0, 0, 0), [], tag="C4")
    names = [f"a{i}" for i in range(12)]
    homes = ["F", "D1", "D2", "D3"]
    for i, (a, d) in enumerate(zip(names, C4_DOMS)):
        R = db.rel(homes[i % 4])
        R.cols[a] = zipf_ranks(_rng(seed, R.name, a), d, 1.0, R.nrows).astype(np.int32)
    return Workload("C4", db, mi_batch(names), {"fact_rows": fact_rows, "attrs": names, "domains": C4_DOMS})


def config5(seed: int = 0, fact_rows: int = 84_000_000, dim_rows=(1_000, 10_000, 100_000, 1_000_000),
            cube_doms=(50, 1_000, 10_000)) -> Workload:
    """BJ configs[4]: data cube + covariance; fact 84M x (4 FK Zipf 1.1 +
    m1..m5 ~ U(0,100) + x1..x3 ~ N(0,1)); D1 1k (A, 10 feats), D2 10k (B, 10),
    D3 100k (C, 10), D4 1M (key only) (reading R12)."""
    fact_feats = [f"m{j}" for j in range(1, 6)] + [f"x{j}" for j in range(1, 4)]

    def dist(seed_, name, n):
        if name.startswith("m"):
            return uniform01(seed_, "F", name, n) * 100.0
        return normal(seed_, "F", name, n)

    db = _snowflake(seed, fact_rows, dim_rows, (10, 10, 10, 0), fact_feats, fact_feat_dist=dist, tag="C5")
    for r, (cname, d) in enumerate(zip("ABC", cube_doms), start=1):
        R = db.rel(f"D{r}")
        R.cols[cname] = _rng(seed, R.name, cname).integers(0, d, R.nrows).astype(np.int32)
    measures = [f"m{j}" for j in range(1, 6)]
    feats = fact_feats + [f"d{r}_{j}" for r in (1, 2, 3) for j in range(1, 11)]
    batch = cube_batch(["A", "B", "C"], measures) + [covar_batch(feats)]
    return Workload("C5", db, batch, {"fact_rows": fact_rows, "features": feats, "measures": measures})


CONFIGS = {"C1": config1, "C2": config2, "C3": config3, "C4": config4, "C5": config5}


# ------------------------------------------------------------------ hand databases
def _i(v):
    return np.asarray(v, dtype=np.int32)


def _d(v):
    return np.asarray(v, dtype=np.float64)


def hand_h1() -> Database:
    """F(a,x), S(a,y); duplicate key 1, dangling a=3."""
    F = Relation("F", {"a": _i([1, 1, 2, 3]), "x": _d([2, 3, 5, 7])})
    S = Relation("S", {"a": _i([1, 1, 2]), "y": _d([10, 20, 30])})
    return Database([F, S], "F", [("F", "S")])


def hand_h2(root: str = "F") -> Database:
    """H2: F(a,b,x), S(a,g), T(b,y); dangling a=2, duplicate b=1. H5 = rooted at S."""
    F = Relation("F", {"a": _i([0, 0, 1, 1, 2]), "b": _i([0, 1, 0, 1, 0]), "x": _d([1, 2, 4, 8, 16])})
    S = Relation("S", {"a": _i([0, 1]), "g": _i([7, 9])})
    T = Relation("T", {"b": _i([0, 1, 1]), "y": _d([0.5, 0.25, 0.75])})
    if root == "F":
        return Database([F, S, T], "F", [("F", "S"), ("F", "T")])
    return Database([F, S, T], "S", [("S", "F"), ("F", "T")])


def hand_h3(root: str = "S1") -> Database:
    """H3: chain S1(X1,X2)-S2(X2,X3)-S3(X3,X4) (the §4.3 shape)."""
    S1 = Relation("S1", {"X1": _i([1, 1, 2]), "X2": _i([1, 2, 1])})
    S2 = Relation("S2", {"X2": _i([1, 2, 2]), "X3": _i([1, 1, 2])})
    S3 = Relation("S3", {"X3": _i([1, 2, 2]), "X4": _i([5, 5, 6])})
    edges = {"S1": [("S1", "S2"), ("S2", "S3")], "S2": [("S2", "S1"), ("S2", "S3")], "S3": [("S3", "S2"), ("S2", "S1")]}
    return Database([S1, S2, S3], root, edges[root])


def hand_h4() -> Database:
    """H4: H1 with S empty."""
    F = Relation("F", {"a": _i([1, 1, 2, 3]), "x": _d([2, 3, 5, 7])})
    S = Relation("S", {"a": _i([]), "y": _d([])})
    return Database([F, S], "F", [("F", "S")])


# ------------------------------------------------------------- random small DBs
def random_db(seed: int, max_rels: int = 5, max_rows: int = 1000, max_dom: int = 50, star: bool = False,
              unique_child_keys: bool = False) -> Database:
    """SPEC-style random acyclic DB: <= max_rels relations, <= max_rows
    rows, key domains <= max_dom.  Each tree edge carries its own int32 join
    attribute j<e>; each relation may carry an int attribute g<r> (domain <= 8)
    and float attributes v<r>_<i>.  star=True: every non-root hangs off the root.
    unique_child_keys=True: children have unique join-key values (PK dims)."""
    rng = _rng(seed, "random_db")
    m = int(rng.integers(1, max_rels + 1))
    names = [f"R{i}" for i in range(m)]
    parent = [-1] + [0 if star else int(rng.integers(0, i)) for i in range(1, m)]
    doms = [int(rng.integers(2, max_dom + 1)) for _ in range(m)]
    rows = [int(rng.integers(0, max_rows + 1)) for _ in range(m)]
    if m > 0:
        rows[0] = max(rows[0], 1)
    cols = [dict() for _ in range(m)]
    for c in range(1, m):
        p = parent[c]
        key = f"j{c}"
        if unique_child_keys:
            rows[c] = min(rows[c], doms[c])
            cols[c][key] = rng.permutation(doms[c])[: rows[c]].astype(np.int32)
        else:
            cols[c][key] = rng.integers(0, doms[c], rows[c]).astype(np.int32)
        cols[p][key] = None  # filled once the parent's row count is fixed
        cols[p].setdefault("_fk", []).append((key, doms[c]))
    for r in range(m):
        n = rows[r]
        for key, dom in cols[r].pop("_fk", []):
            # a few dangling values (dom + 1 is never a child key)
            v = rng.integers(0, dom + 1, n)
            cols[r][key] = v.astype(np.int32)
        if rng.random() < 0.7:
            cols[r][f"g{r}"] = rng.integers(0, int(rng.integers(1, 9)), n).astype(np.int32)
        for i in range(int(rng.integers(0, 3))):
            cols[r][f"v{r}_{i}"] = np.round(rng.standard_normal(n) * 4) / 4  # dyadic values
    rels = [Relation(names[r], cols[r]) for r in range(m)]
    edges = [(names[parent[c]], names[c]) for c in range(1, m)]
    return Database(rels, names[0], edges)


def attributes(db: Database) -> dict:
    """attr name -> dtype kind ('i' or 'f')."""
    out = {}
    for r in db.relations:
        for c, v in r.cols.items():
            out[c] = "i" if v.dtype == np.int32 else "f"
    return out


def random_batch(seed: int, db: Database, n_queries: int = 3, max_udafs: int = 4, groupby_ok=None) -> list:
    """Random batch: group-by over int attributes (optionally filtered), UDAFs as
    random sums of products of const/ident/predicate factors."""
    rng = _rng(seed, "random_batch")
    attrs = attributes(db)
    ints = sorted(a for a, k in attrs.items() if k == "i")
    allat = sorted(attrs)
    gb_pool = [a for a in ints if groupby_ok is None or groupby_ok(a)]
    batch = []
    for q in range(n_queries):
        ngb = int(rng.integers(0, min(2, len(gb_pool)) + 1)) if gb_pool else 0
        gb = list(rng.choice(gb_pool, ngb, replace=False)) if ngb else []
        udafs = []
        for _ in range(int(rng.integers(1, max_udafs + 1))):
            prods = []
            for _ in range(int(rng.integers(0, 3))):
                fs = []
                for _ in range(int(rng.integers(0, 4))):
                    kind = int(rng.choice([F_CONST, F_IDENT, F_IDENT, F_LT, F_LE, F_GT, F_GE, F_EQ, F_NE]))
                    if kind == F_CONST:
                        fs.append(Factor(F_CONST, None, float(rng.integers(-2, 3)) / 2))
                    else:
                        a = str(rng.choice(allat))
                        param = float(rng.integers(-4, 5)) / 2 if attrs[a] == "f" else float(rng.integers(0, 10))
                        fs.append(Factor(kind, a, param))
                prods.append(Product(float(rng.integers(-3, 4)) / 2 or 1.0, tuple(fs)))
            udafs.append(prods)
        batch.append(Query([str(g) for g in gb], udafs, name=f"rq{q}"))
    return batch
