"""Parity of the count path (counts.cu, §8 row (e)): COUNT GROUP BY over one or two
attributes of the root and of primary-key leaves (the Chow-Liu / mutual-information batch
of BASELINE.json configs[3]), dimension-only queries finished through the per-key row
counts, constant UDAFs, COUNT, skewed and ragged inputs, against the oracle."""
import numpy as np
import pytest

import oracle
import synth
from _parity import assert_parity, run_gpu
from synth import Product, Query

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("runs,pack", [(None, "1"), ("0", "1"), ("1", "1"), (None, "0")])
@pytest.mark.parametrize("n", [1, 31, 33, 5000, 40_011])
def test_counts_config4_shape(n, runs, pack, monkeypatch):
    """runs: cross-dimension tables counted once per run segment at the first two sort positions
    (default), never ("0"), or at every position ("1"; LMFAO_CNT_RUNS); pack=0: dimension codes
    gathered one attribute at a time (LMFAO_CNT_PACK)."""
    if runs is not None:
        monkeypatch.setenv("LMFAO_CNT_RUNS", runs)
    monkeypatch.setenv("LMFAO_CNT_PACK", pack)
    w = synth.config4(fact_rows=n, dim_rows=(40, 300, 2000))
    gpu, info = run_gpu(w.db, w.batch, info=True)
    assert info["fast_path"] and info["fast_path"]["kind"] == "counts", info
    assert_parity(gpu, oracle.evaluate(w.db, w.batch), w.batch)


def test_counts_constants_and_mixed_levels():
    w = synth.config4(fact_rows=20_000, dim_rows=(30, 200, 1500))
    batch = [Query(["a0", "a1"], [[Product(2.0, ())], [Product(1.0, ()), Product(-0.5, ())]]),
             Query(["a5", "a9"], [[Product(1.0, ())]]),       # both in D1: dimension side
             Query(["a11"], [[Product(3.0, ())]]),             # single dim attribute
             Query(["a7", "a2"], [[Product(1.0, ())]]),       # two different dims
             Query(["a4"], [[Product(1.0, ())]]),
             Query([], [[Product(1.0, ())], [Product(4.0, ())]])]
    gpu, info = run_gpu(w.db, batch, info=True)
    assert info["fast_path"]["kind"] == "counts"
    assert_parity(gpu, oracle.evaluate(w.db, batch), batch)


def test_counts_matches_generic(monkeypatch):
    w = synth.config4(fact_rows=60_000, dim_rows=(40, 300, 2000))
    g1 = run_gpu(w.db, w.batch)
    monkeypatch.setenv("LMFAO_GENERIC_ONLY", "1")
    g2 = run_gpu(w.db, w.batch)
    for (k1, v1, c1), (k2, v2, c2) in zip(g1, g2):
        assert np.array_equal(k1, k2) and np.array_equal(c1, c2) and np.array_equal(v1, v2)


@pytest.mark.parametrize("nparts", [2, 3])
def test_counts_sharded(nparts):
    w = synth.config4(fact_rows=20_011, dim_rows=(30, 200, 1500))
    ref = oracle.evaluate(w.db, w.batch)
    parts = [run_gpu(w.db, w.batch, shard=(p, nparts)) for p in range(nparts)]
    q = len(w.batch) - 1  # COUNT
    assert sum(int(p[q][2][0]) for p in parts) == int(ref[q].counts[0])
    # a root x dimension pair: per-cell counts of the shards add up to the oracle's
    qi = 0
    tot = {}
    for p in parts:
        k, v, c = p[qi]
        for kk, cc in zip(map(tuple, k.astype(np.int64)), c):
            tot[kk] = tot.get(kk, 0) + int(cc)
    assert tot == {tuple(kk): int(cc) for kk, cc in zip(ref[qi].keys, ref[qi].counts)}


def _wide_star(n, ndims, attrs_per_rel, seed=5):
    """A star with `ndims` primary-key leaves and `attrs_per_rel` Zipf categoricals in the root
    and in every dimension (wider than C4: the per-warp code rows of k_cnt_rows no longer fit
    beside 1024 threads, so the planner takes fewer threads and a smaller shared budget)."""
    db = synth._snowflake(seed, n, tuple(20 + 37 * r for r in range(ndims)), (0,) * ndims, [], tag="W")
    names = []
    for ri, rel in enumerate(["F"] + [f"D{r}" for r in range(1, ndims + 1)]):
        R = db.rel(rel)
        for j in range(attrs_per_rel):
            a = f"c{ri}_{j}"
            R.cols[a] = synth.zipf_ranks(synth._rng(seed, rel, a), 3 + 11 * j + 5 * ri, 1.0, R.nrows).astype(np.int32)
            names.append(a)
    return db, names


@pytest.mark.parametrize("cells", [None, "0", "700"])
def test_counts_wide_batch_smem_budgets(monkeypatch, cells):
    """24 attributes over 8 relations (the kernel's maxima): every pair, single and COUNT,
    with the default shared budget (capped by the planner), none, and a small one."""
    if cells is not None:
        monkeypatch.setenv("LMFAO_CNT_SMEM_CELLS", cells)
    db, names = _wide_star(9_001, 7, 3)
    assert len(names) == 24
    batch = synth.mi_batch(names)  # 276 pairs, 24 singles, COUNT
    gpu, info = run_gpu(db, batch, info=True)
    assert info["fast_path"]["kind"] == "counts", info
    assert_parity(gpu, oracle.evaluate(db, batch), batch)


@pytest.mark.parametrize("views,cap,every", [("0", None, False), ("1", None, False), ("1", "2000", False),
                                             ("1", None, True)])
def test_counts_views(monkeypatch, views, cap, every):
    """Pair queries finished from shared views V_D[k][b] (LMFAO_CNT_VIEWS):
    none, the default choice, only the small views (LMFAO_CNT_VIEW_CELLS: the rest per row), and
    every candidate (any table size, views keyed by any level)."""
    monkeypatch.setenv("LMFAO_CNT_VIEWS", views)
    if cap is not None:
        monkeypatch.setenv("LMFAO_CNT_VIEW_CELLS", cap)
        monkeypatch.setenv("LMFAO_CNT_VIEW_MIN", "0")
    if every:
        monkeypatch.setenv("LMFAO_CNT_VIEW_MIN", "0")
        monkeypatch.setenv("LMFAO_CNT_VIEW_POS", "8")
    w = synth.config4(fact_rows=50_003, dim_rows=(40, 300, 2000))
    gpu, info = run_gpu(w.db, w.batch, info=True)
    fp = info["fast_path"]
    assert fp["kind"] == "counts", info
    if views == "0":
        assert fp["views"] == 0
    else:
        assert fp["views"] > 0 and fp["view_queries"] >= 2 * fp["views"], fp
        assert fp["row_queries"] == 60 - fp["view_queries"] + fp["views"], fp
    assert_parity(gpu, oracle.evaluate(w.db, w.batch), w.batch)
