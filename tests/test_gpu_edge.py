"""Degenerate inputs through every specialised path (cov.cu, gram.cu, rt.cu, counts.cu, cube.cu) and
the view kernels: a root whose rows all dangle (empty join), a single-row root, dimensions
with a single key, and a root that shrinks to one 32-row block after dropping dangling rows."""
import numpy as np
import pytest

import oracle
import synth
from _parity import assert_parity, run_gpu

pytestmark = pytest.mark.gpu


def star(n, dim_rows, dangle_all=False, seed=0, nf=3, df=(2, 3, 4)):
    rng = np.random.default_rng(seed)
    F, dims = {}, []
    for r, (nr, f) in enumerate(zip(dim_rows, df), start=1):
        keys = np.arange(nr, dtype=np.int32) * 3
        cols = {f"k{r}": keys, f"c{r}": rng.integers(0, 4, nr).astype(np.int32)}
        for j in range(f):
            cols[f"d{r}_{j}"] = rng.standard_normal(nr)
        dims.append(synth.Relation(f"D{r}", cols))
        fk = keys[rng.integers(0, nr, n)] if nr else np.zeros(n, np.int32)
        F[f"k{r}"] = (fk + 1 if dangle_all else fk).astype(np.int32)
    for j in range(nf):
        F[f"x{j}"] = rng.standard_normal(n)
    F["y"] = rng.standard_normal(n)
    F["g"] = rng.integers(0, 3, n).astype(np.int32)
    db = synth.Database([synth.Relation("F", F)] + dims, "F", [("F", d.name) for d in dims])
    feats = [f"x{j}" for j in range(nf)] + [f"d{r}_{j}" for r, f in enumerate(df, 1) for j in range(f)]
    return db, feats


def batches(feats):
    return {
        "cov": [synth.covar_batch(feats)],
        "rt": synth.rt_batch(feats[:4], "y", ["g", "c1", "c3"], synth.thresholds_c3()[::5]),
        "counts": [synth.Query(["g", "c2"], [[synth.Product(1.0, ())]]), synth.Query(["c1"], [[synth.Product(1.0, ())]]),
                   synth.Query([], [[synth.Product(1.0, ())]])],
        "cube": [synth.Query(["c1"], [[synth.Product(1.0, (synth.ident("x0"),))], [synth.Product(1.0, ())]]),
                 synth.Query(["c1", "c3"], [[synth.Product(2.0, (synth.ident("y"),))]]),
                 synth.Query(["g", "c2"], [[synth.Product(1.0, (synth.ident("x1"),)), synth.Product(-3.0, ())]]),
                 synth.Query([], [[synth.Product(1.0, (synth.ident("y"),))]])],
    }


@pytest.mark.parametrize("kind", ["cov", "rt", "counts", "cube"])
@pytest.mark.parametrize("case", ["all_dangling", "one_row", "single_keys", "one_block"])
def test_degenerate(kind, case):
    if case == "all_dangling":
        db, feats = star(5000, (20, 30, 40), dangle_all=True)
    elif case == "one_row":
        db, feats = star(1, (20, 30, 40))
    elif case == "single_keys":
        db, feats = star(3000, (1, 1, 1))
    else:
        db, feats = star(29, (20, 30, 40), seed=3)
    batch = batches(feats)[kind]
    gpu, info = run_gpu(db, batch, info=True)
    ref = oracle.evaluate(db, batch)
    assert_parity(gpu, ref, batch)


def test_reset_batch_reuses_prepared_relations():
    """lmfao_reset_batch: STATE error before prepare; afterwards batches of different shapes
    (covariance, counts, cube, rt) over the same prepared data all match the oracle."""
    from paper_1906_08687_b200 import lmfao
    db, feats = star(4000, (20, 30, 40), seed=5)
    e = lmfao.Engine()
    try:
        for r in db.relations:
            e.add_relation(r.name, r.cols)
        with pytest.raises(lmfao.LmfaoError) as ei:
            e.reset_batch()
        assert ei.value.name == "LMFAO_ERR_STATE"
        e.set_join_tree(db.root, db.edges)
        e.prepare()
        for kind in ["cov", "counts", "cube", "rt", "cov"]:
            batch = batches(feats)[kind]
            qids = [e.add_query(q.groupby, q.udafs) for q in batch]
            e.plan()
            e.run()
            e.run()
            got = [e.fetch(q) for q in qids]
            assert_parity(got, oracle.evaluate(db, batch), batch)
            e.reset_batch()
    finally:
        e.close()
