"""NEXT-2 batches at C2 scale (10M rows): categorical covariance (C2's 38 features plus three
categoricals: Covar(X_j; X_k) and Covar(X_j, X_k; 1)) and degree-2 polynomial aggregates over
four features; lmfao_run time and the path the planner picked.  usage: python tools/time_next2.py"""
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1906_08687_b200 import lmfao  # noqa: E402
from synth import Product, Query, ident  # noqa: E402

w = synth.config2()
rng = np.random.default_rng(0)
F = w.db.rel("F")
F.cols["cf"] = rng.integers(0, 6, F.nrows).astype(np.int32)
for r, d in ((1, 4), (3, 9)):
    R = w.db.rel(f"D{r}")
    R.cols[f"cat{r}"] = rng.integers(0, d, R.nrows).astype(np.int32)
feats = w.meta["features"]
cats = ["cf", "cat1", "cat3"]
catcov = [synth.covar_batch(feats)]
for k in cats:
    catcov.append(Query([k], [[Product(1.0, ())]] + [[Product(1.0, (ident(j),))] for j in feats]))
for a, b in itertools.combinations(cats, 2):
    catcov.append(Query([a, b], [[Product(1.0, ())]]))
pf = ["x1", "x2", "d1_1", "d3_1"]
mons = [()] + [(f,) for f in pf] + list(itertools.combinations_with_replacement(pf, 2))
poly = [Query([], [[Product(1.0, tuple(ident(a) for a in m1 + m2))] for i, m1 in enumerate(mons) for m2 in mons[i:]])]
torch.cuda.set_stream(torch.cuda.Stream())
cols = {r.name: {c: torch.from_numpy(v).cuda() for c, v in r.cols.items()} for r in w.db.relations}
sp = torch.cuda.current_stream().cuda_stream
for name, batch, env in (("categorical covariance", catcov, None), ("degree-2 polynomial", poly, None),
                         ("degree-2 polynomial, interpreted", poly, "LMFAO_NO_POLY")):
    if env:
        os.environ[env] = "1"
    e = lmfao.Engine()
    lmfao.load(e, w.db, batch, columns=cols)
    e.plan()
    e.run(sp)
    e.run(sp)
    torch.cuda.synchronize()
    s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        e.run(sp)
    t.record()
    torch.cuda.synchronize()
    print(json.dumps({"batch": name, "fact_rows": F.nrows, "aggregates": synth.n_aggregates(batch),
                      "run_ms": s.elapsed_time(t) / 5, "plan": e.plan_info().get("fast_path")}), flush=True)
    e.close()
    if env:
        del os.environ[env]
