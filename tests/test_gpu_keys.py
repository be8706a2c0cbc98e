"""Two-attribute join keys ("multi-attribute join keys (Favorita's
(date, store))"): an edge sharing two int32 attributes is matched on the pair — a dictionary
over the child's distinct pairs at prepare, the parent's pairs looked up in it (dangling
pairs drop rows).  Parity against the oracle, which matches the shared attributes directly."""
import numpy as np
import pytest

import oracle
import synth
from _parity import assert_parity, run_gpu

pytestmark = pytest.mark.gpu


def favorita_like(seed, n, dangle=0.0, dup=False):
    """Sales(date, store, item, units, onpromo) with Oil(date), Stores(store), Items(item) and a
    two-attribute edge to Transactions(date, store)."""
    rng = np.random.default_rng(seed)
    dates = np.arange(100, dtype=np.int32) * 3 - 50
    stores = np.arange(12, dtype=np.int32) + 7
    items = np.arange(300, dtype=np.int32)
    d, s = np.meshgrid(dates, stores, indexing="ij")
    pairs = np.stack([d.ravel(), s.ravel()], 1)
    keep = rng.random(len(pairs)) > 0.2  # not every (date, store) has transactions
    if dup:  # a many-to-many edge: some pairs twice
        keep = np.concatenate([keep, rng.random(len(pairs)) > 0.9])
        pairs = np.concatenate([pairs, pairs])
    pairs = pairs[keep]
    perm = rng.permutation(len(pairs))
    tr = synth.Relation("T", {"date": pairs[perm, 0].astype(np.int32), "store": pairs[perm, 1].astype(np.int32),
                              "trans": rng.standard_normal(len(pairs)), "tcat": rng.integers(0, 4, len(pairs)).astype(np.int32)})
    oil = synth.Relation("O", {"date": dates, "price": rng.standard_normal(len(dates))})
    st = synth.Relation("S", {"store": stores, "cluster": rng.integers(0, 5, len(stores)).astype(np.int32),
                              "sz": rng.standard_normal(len(stores))})
    it = synth.Relation("I", {"item": items, "perish": rng.standard_normal(len(items))})
    sales = {"date": dates[rng.integers(0, len(dates), n)], "store": stores[rng.integers(0, len(stores), n)],
             "item": items[rng.integers(0, len(items), n)]}
    if dangle:
        m = rng.random(n) < dangle
        sales["store"] = np.where(m, 999, sales["store"]).astype(np.int32)
    sales["units"] = rng.standard_normal(n)
    sales["promo"] = rng.integers(0, 2, n).astype(np.int32)
    F = synth.Relation("F", sales)
    # T is the child of F on (date, store); O and S hang below T? No: O, S, I are children of F
    # through date / store / item — the running intersection holds since T shares both with F.
    return synth.Database([F, tr, oil, st, it], "F", [("F", "T"), ("F", "O"), ("F", "S"), ("F", "I")])


def cov_batch():
    return [synth.covar_batch(["units", "trans", "price", "sz"])]  # <= 3 featured levels (cov.cu)


def group_batch():
    P, I = synth.Product, synth.ident
    return [synth.Query(["tcat"], [[P(1.0, (I("units"),))], [P(1.0, ())]]),
            synth.Query(["promo", "cluster"], [[P(1.0, (I("trans"),))]]),
            synth.Query([], [[P(1.0, (I("units"), I("trans")))], [P(1.0, ())]])]


@pytest.mark.parametrize("n", [1, 500, 40_000])
def test_pair_key_covariance(n):
    db = favorita_like(1, n)
    batch = cov_batch()
    gpu, info = run_gpu(db, batch, info=True)
    assert info["fast_path"]["kind"] == "cov", info["fast_path"]
    assert_parity(gpu, oracle.evaluate(db, batch), batch)


def test_pair_key_dangling_and_groups():
    db = favorita_like(2, 30_000, dangle=0.1)
    batch = group_batch()
    ref = oracle.evaluate(db, batch)
    assert int(ref[2].counts[0]) < 30_000
    assert_parity(run_gpu(db, batch), ref, batch)


def test_pair_key_many_to_many():
    """Duplicate (date, store) pairs in T: the generic path's view multiplicities."""
    db = favorita_like(3, 20_000, dup=True)
    batch = cov_batch() + group_batch()[1:]  # (group-bys on T's own attributes need a unique key, v1)
    assert_parity(run_gpu(db, batch), oracle.evaluate(db, batch), batch)


def three_attr_db(seed, n, dangle=0.0, dup=False):
    """Sales(date, store, item, units) with an inventory child Inv(date, store, item, stock, cat)
    joined on the three attributes (keys of more than two attributes: a chain of pair
    dictionaries at prepare), plus Oil(date) and Items(item) on one attribute each."""
    rng = np.random.default_rng(seed)
    dates = np.arange(20, dtype=np.int32) * 7 - 30
    stores = np.arange(6, dtype=np.int32) + 100
    items = np.arange(40, dtype=np.int32) * 2
    d, s, i = np.meshgrid(dates, stores, items, indexing="ij")
    trip = np.stack([d.ravel(), s.ravel(), i.ravel()], 1)
    trip = trip[rng.random(len(trip)) > 0.3]  # not every triple stocked
    if dup:
        trip = np.concatenate([trip, trip[rng.random(len(trip)) > 0.9]])
    trip = trip[rng.permutation(len(trip))]
    inv = synth.Relation("V", {"date": trip[:, 0].astype(np.int32), "store": trip[:, 1].astype(np.int32),
                               "item": trip[:, 2].astype(np.int32), "stock": rng.standard_normal(len(trip)),
                               "vcat": rng.integers(0, 3, len(trip)).astype(np.int32)})
    oil = synth.Relation("O", {"date": dates, "price": rng.standard_normal(len(dates))})
    it = synth.Relation("I", {"item": items, "perish": rng.standard_normal(len(items))})
    sales = {"date": dates[rng.integers(0, len(dates), n)], "store": stores[rng.integers(0, len(stores), n)],
             "item": items[rng.integers(0, len(items), n)]}
    if dangle:
        sales["item"] = np.where(rng.random(n) < dangle, 7, sales["item"]).astype(np.int32)  # odd: no such item
    sales["units"] = rng.standard_normal(n)
    F = synth.Relation("F", sales)
    return synth.Database([F, inv, oil, it], "F", [("F", "V"), ("F", "O"), ("F", "I")])


@pytest.mark.parametrize("n,dangle,dup", [(1, 0.0, False), (3_000, 0.0, False), (40_000, 0.05, False),
                                          (20_000, 0.0, True)])
def test_three_attribute_key(n, dangle, dup):
    db = three_attr_db(4, n, dangle, dup)
    P, I = synth.Product, synth.ident
    batch = [synth.covar_batch(["units", "stock", "price", "perish"]),
             synth.Query(["date"], [[P(1.0, (I("stock"),))], [P(1.0, ())]])]
    if not dup:  # a group-by on the child's own attribute needs its key unique at this root
        batch.append(synth.Query(["vcat", "store"], [[P(1.0, (I("units"), I("stock")))]]))
    assert_parity(run_gpu(db, batch), oracle.evaluate(db, batch), batch)
