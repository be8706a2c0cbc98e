"""Parity of the view build (b) for many-to-many children: a child sorted by its join key
with Zipf-hot keys whose runs span many 32-row blocks and warp ranges (the carried-run
path), cold keys (runs inside a block), through both view kernels (k_view_lin: identity
slots; k_view_build: interpreted slots with predicates and a grandchild)."""
import numpy as np
import pytest

import oracle
import synth
from _parity import assert_parity, run_gpu
from synth import F_GT, F_LE, Factor, Product, Query, ident

pytestmark = pytest.mark.gpu


def m2m_db(seed, n_child, n_keys, s, grandchild=False):
    rng = np.random.default_rng(seed)
    keys = np.arange(n_keys, dtype=np.int32)
    D = {"k": keys[synth.zipf_ranks(rng, n_keys, s, n_child)].astype(np.int32),
         "d0": rng.standard_normal(n_child), "d1": np.round(rng.standard_normal(n_child) * 4) / 4,
         "e": rng.integers(0, 7, n_child).astype(np.int32)}
    F = {"k": rng.integers(0, n_keys + 3, 3000).astype(np.int32), "x": rng.standard_normal(3000),
         "g": rng.integers(0, 5, 3000).astype(np.int32)}
    rels = [synth.Relation("F", F), synth.Relation("D", D)]
    edges = [("F", "D")]
    if grandchild:
        D["j"] = rng.integers(0, 40, n_child).astype(np.int32)
        rels.append(synth.Relation("G", {"j": rng.integers(0, 40, 100).astype(np.int32),
                                         "gv": rng.standard_normal(100)}))
        edges.append(("D", "G"))
    return synth.Database(rels, "F", edges)


@pytest.mark.parametrize("n_child,n_keys,s", [(200_000, 500, 1.1), (150_011, 50_000, 1.1), (70_000, 20, 0.0),
                                               (33, 4, 1.0)])
def test_view_lin_long_and_short_runs(n_child, n_keys, s):
    db = m2m_db(1, n_child, n_keys, s)
    batch = [synth.covar_batch(["x", "d0", "d1"]), Query(["g"], [[Product(1.0, (ident("d0"),))],
                                                               [Product(1.0, (ident("x"), ident("d1")))]])]
    assert_parity(run_gpu(db, batch), oracle.evaluate(db, batch), batch)


@pytest.mark.parametrize("grandchild", [False, True])
def test_view_interpreted_predicates(grandchild):
    db = m2m_db(2, 120_000, 300, 1.2, grandchild)
    udafs = [[Product(1.0, (Factor(F_LE, "d1", 0.25),))], [Product(1.0, (ident("d0"), Factor(F_GT, "e", 2.0)))],
             [Product(2.0, (ident("x"), Factor(F_LE, "d0", 0.0)))]]
    if grandchild:
        udafs.append([Product(1.0, (ident("gv"), ident("d0")))])
    batch = [Query([], udafs), Query(["g"], udafs[:2])]
    assert_parity(run_gpu(db, batch), oracle.evaluate(db, batch), batch)


@pytest.mark.parametrize("fast", ["1", "0"])
@pytest.mark.parametrize("n_child,n_keys,s,nfeat", [(300_007, 2_000, 1.1, 10), (90_000, 30_000, 1.1, 15),
                                                     (50_000, 3, 0.0, 2), (64, 5, 1.0, 1), (1, 1, 0.0, 4)])
def test_view_lin_fast_count_and_columns(fast, n_child, n_keys, s, nfeat, monkeypatch):
    """The register path of k_view_lin (every slot the count or one fp64 column, <= 16 slots:
    the (b) view bench's shape) and the generic one (LMFAO_VIEW_FAST=0) against the oracle:
    runs through many blocks and warp ranges, runs inside a block, ragged ends."""
    rng = np.random.default_rng(7)
    keys = np.arange(n_keys, dtype=np.int32)
    D = {"k": keys[synth.zipf_ranks(rng, n_keys, s, n_child)].astype(np.int32)}
    for j in range(nfeat):
        D[f"d{j}"] = rng.standard_normal(n_child)
    F = {"k": rng.integers(0, n_keys + 2, 2_000).astype(np.int32), "x": rng.standard_normal(2_000),
         "g": rng.integers(0, 4, 2_000).astype(np.int32)}
    db = synth.Database([synth.Relation("F", F), synth.Relation("D", D)], "F", [("F", "D")])
    sums = [[Product(1.0, (ident(f"d{j}"),))] for j in range(nfeat)]
    batch = [Query([], [[Product(1.0, ())]] + sums), Query(["g"], sums[:2] + [[Product(1.0, (ident("x"),))]])]
    monkeypatch.setenv("LMFAO_VIEW_FAST", fast)
    assert_parity(run_gpu(db, batch, runs=2), oracle.evaluate(db, batch), batch)
