"""Covariance batches over snowflakes deeper than a star ("depth > 1
snowflakes at scale"; PAPER.md's Retailer is Inventory → Location → Census/Weather):
with every non-root relation unique-keyed, a root row joins one row of each, so the cov.cu
scan gathers a dimension key's whole subtree of features through composed foreign keys
(dangling keys anywhere drop rows at prepare).  Parity against the oracle."""
import numpy as np
import pytest

import oracle
import synth
from _parity import assert_parity, run_gpu

pytestmark = pytest.mark.gpu


def snowflake(seed, n, dangle=False):
    rng = np.random.default_rng(seed)

    def rel(name, key, nk, feats, fks=()):
        cols = {key: (np.arange(nk, dtype=np.int32) * 7 + 3)}
        for f in feats:
            cols[f] = rng.standard_normal(nk)
        for fk, target_keys in fks:
            v = target_keys[rng.integers(0, len(target_keys), nk)]
            if dangle:
                v = v.copy()
                v[rng.random(nk) < 0.05] = -5  # references a missing key
            cols[fk] = v.astype(np.int32)
        return synth.Relation(name, cols)

    G2 = rel("G2", "g2", 15, ["gf1", "gf2"])
    E2 = rel("E2", "e2", 60, ["ef1", "ef2", "ef3"], [("g2", G2.cols["g2"])])
    E1 = rel("E1", "e1", 40, ["hf1", "hf2"])
    D1 = rel("D1", "k1", 120, ["a1", "a2", "a3"], [("e1", E1.cols["e1"])])
    D2 = rel("D2", "k2", 900, ["b1", "b2"], [("e2", E2.cols["e2"])])
    D3 = rel("D3", "k3", 3000, ["c1", "c2", "c3", "c4"])
    F = {}
    for D, key in ((D1, "k1"), (D2, "k2"), (D3, "k3")):
        F[key] = synth.zipf_fk(seed, "F", key, D.cols[key], 1.1, n)
    for j in range(1, 5):
        F[f"x{j}"] = rng.standard_normal(n)
    rels = [synth.Relation("F", F), D1, D2, D3, E1, E2, G2]
    edges = [("F", "D1"), ("F", "D2"), ("F", "D3"), ("D1", "E1"), ("D2", "E2"), ("E2", "G2")]
    feats = ["x1", "x2", "x3", "x4", "a1", "a2", "a3", "hf1", "hf2", "b1", "b2", "ef1", "ef2", "ef3", "gf1", "gf2",
             "c1", "c2", "c3", "c4"]
    return synth.Database(rels, "F", edges), feats


@pytest.mark.parametrize("n", [1, 33, 4_097, 60_000])
def test_snowflake_covariance_on_the_scan(n):
    db, feats = snowflake(1, n)
    batch = [synth.covar_batch(feats)]
    gpu, info = run_gpu(db, batch, info=True)
    assert info["fast_path"]["kind"] == "cov", info["fast_path"]
    assert_parity(gpu, oracle.evaluate(db, batch), batch)


def test_snowflake_with_dangling_keys():
    db, feats = snowflake(2, 30_000, dangle=True)
    batch = [synth.covar_batch(feats[:6] + feats[9:14])]
    gpu, info = run_gpu(db, batch, info=True)
    assert info["fast_path"]["kind"] == "cov", info["fast_path"]
    ref = oracle.evaluate(db, batch)
    assert 0 < int(ref[0].counts[0]) < 30_000
    assert_parity(gpu, ref, batch)


def test_snowflake_matches_generic(monkeypatch):
    db, feats = snowflake(3, 20_000)
    batch = [synth.covar_batch(feats)]
    g1 = run_gpu(db, batch)
    monkeypatch.setenv("LMFAO_GENERIC_ONLY", "1")
    g2 = run_gpu(db, batch)
    assert np.array_equal(g1[0][2], g2[0][2])
    assert np.allclose(g1[0][1], g2[0][1], rtol=1e-11, atol=1e-9)
