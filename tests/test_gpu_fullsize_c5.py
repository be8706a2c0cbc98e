"""Parity at BASELINE.json configs[4]'s full size (C5: 84M fact rows, the data cube over
A/B/C with 5 measures + the 38-feature covariance batch), stratified so the oracle
finishes in about a minute on the host cores while every part of the result is covered:

  * covariance: three aggregates of every block — COUNT, Σ fact / D1 / D2 / D3 feature,
    fact⊗fact, fact⊗D_r, D_r⊗D_r and D_r⊗D_q — recomputed over the whole 84M-row join;
  * cube: every one of the 8 cuboids, on a sample of its groups.  The sample is a
    selection: the dimension rows whose cube attributes take sampled values (values of
    randomly drawn fact rows, so hot and cold groups both appear), and the fact rows that
    join them.  Over that restricted database the oracle's groups are exactly the GPU's
    groups whose keys lie in the sampled value sets (selections commute with the join).
The GPU evaluates the whole batch once, over the whole database, as bench.py/time_configs do.
"""
import numpy as np
import pytest

import oracle
import synth
from _parity import run_gpu
from _udaf import float_close

pytestmark = pytest.mark.gpu

N5 = 84_000_000


@pytest.fixture(scope="module")
def c5():
    w = synth.config5()
    gpu = run_gpu(w.db, w.batch)
    return w, gpu


def _blocks(feats):
    fact = [f for f in feats if not f.startswith("d")]
    dims = {r: [f for f in feats if f.startswith(f"d{r}_")] for r in (1, 2, 3)}
    groups = {"count": [()], "lin_fact": [(a,) for a in fact]}
    for r in (1, 2, 3):
        groups[f"lin_D{r}"] = [(a,) for a in dims[r]]
    groups["fact_fact"] = [(a, b) for i, a in enumerate(fact) for b in fact[i:]]
    for r in (1, 2, 3):
        groups[f"fact_D{r}"] = [(a, b) for a in fact for b in dims[r]]
        groups[f"D{r}_D{r}"] = [(a, b) for i, a in enumerate(dims[r]) for b in dims[r][i:]]
    for r, q in ((1, 2), (1, 3), (2, 3)):
        groups[f"D{r}_D{q}"] = [(a, b) for a in dims[r] for b in dims[q]]
    return groups


def test_c5_full_covariance_every_block(c5):
    w, gpu = c5
    qi = len(w.batch) - 1
    feats = w.meta["features"]
    # the covariance batch's UDAF order (synth.covar_batch): 1, x_i, then x_i*x_j for i <= j
    order = [()] + [(a,) for a in feats] + [(a, b) for i, a in enumerate(feats) for b in feats[i:]]
    pos = {t: j for j, t in enumerate(order)}
    rng = np.random.default_rng(5)
    idx = []
    for name, terms in _blocks(feats).items():
        pick = rng.choice(len(terms), size=min(3, len(terms)), replace=False)
        idx += [pos[terms[p]] for p in pick]
    idx = sorted(idx)
    assert len(idx) >= 40
    q = synth.Query([], [w.batch[qi].udafs[i] for i in idx])
    ref = oracle.evaluate(w.db, [q], threads=0)[0]
    k, v, c = gpu[qi]
    assert int(c[0]) == N5 == int(ref.counts[0])
    ok = float_close(v[:, idx], ref.vals, ref.absmass)
    assert ok.all(), (np.array(idx)[~ok[0]], v[:, idx][~ok], ref.vals[~ok])


def _restrict(w, sets):
    """The database restricted to dimension rows whose cube attribute lies in sets[attr],
    and to the fact rows joining them (a selection; no arithmetic of the method)."""
    db = w.db
    F = db.rel(db.root)
    keep = np.ones(F.nrows, dtype=bool)
    rels = []
    for R in db.relations:
        if R.name == db.root:
            continue
        attr = next((a for a in ("A", "B", "C") if a in R.cols), None)
        if attr is None or attr not in sets:
            rels.append(R)
            continue
        m = np.isin(R.cols[attr], np.asarray(sorted(sets[attr]), dtype=np.int32))
        Rr = synth.Relation(R.name, {c: v[m] for c, v in R.cols.items()})
        key = next(c for c in R.cols if c in F.cols)
        keep &= np.isin(F.cols[key], Rr.cols[key])
        rels.append(Rr)
    Fr = synth.Relation(F.name, {c: v[keep] for c, v in F.cols.items()})
    return synth.Database([Fr] + rels, db.root, db.edges), int(keep.sum())


@pytest.mark.parametrize("cub", range(8))
def test_c5_full_cuboid_sampled_groups(c5, cub):
    w, gpu = c5
    q = w.batch[cub]
    gb = list(q.groupby)
    db = w.db
    F = db.rel(db.root)
    rng = np.random.default_rng(100 + cub)
    # sampled values: the cube attributes of randomly drawn fact rows (hot and cold groups)
    nval = {1: 3, 2: 12, 3: 40}.get(len(gb), 0)
    rows = rng.integers(0, F.nrows, size=nval)
    sets = {}
    for a in gb:
        R = next(r for r in db.relations if a in r.cols)
        key = next(c for c in R.cols if c in F.cols)
        order = np.argsort(R.cols[key])
        pos = order[np.searchsorted(R.cols[key], F.cols[key][rows], sorter=order)]
        sets[a] = set(int(x) for x in R.cols[a][pos])
    sub, nrows = _restrict(w, sets) if gb else (db, F.nrows)
    ref = oracle.evaluate(sub, [q], threads=0)[0]
    k, v, c = gpu[cub]
    sel = np.ones(len(k), dtype=bool)
    for j, a in enumerate(gb):
        sel &= np.isin(k[:, j], np.asarray(sorted(sets[a]), dtype=np.int32))
    assert sel.sum() == len(ref.keys) > 0
    assert np.array_equal(k[sel].astype(np.int64), ref.keys)
    assert np.array_equal(c[sel], ref.counts)
    assert int(c.sum()) == N5
    ok = float_close(v[sel], ref.vals, ref.absmass)
    assert ok.all(), (gb, np.argwhere(~ok)[:5])
