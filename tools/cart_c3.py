"""Grow the paper's regression tree (depth 4, min split 1000, 20 thresholds per feature,
P:1911-1916) over C3's 10M-row snowflake with one rt.cu node batch per tree node
(apps.regression_tree); prints nodes, wall time and the per-node average.
usage: python tools/cart_c3.py [fact_rows]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1906_08687_b200 import apps, lmfao  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
w = synth.config3(fact_rows=rows)
feats = w.meta["features"]
cols = {r.name: {c: torch.from_numpy(v).cuda() for c, v in r.cols.items()} for r in w.db.relations}
e = lmfao.Engine()
lmfao.load(e, w.db, [], columns=cols)
torch.cuda.synchronize()


def count(n):
    return 1 + (count(n["left"]) + count(n["right"]) if "feature" in n else 0)


trees = {}
for dynamic in (True, False, True):  # dynamic path conditions (one plan) vs one plan per node
    t0 = time.perf_counter()
    tree = apps.regression_tree(e, feats, "y", synth.thresholds_c3(), max_depth=4, min_split=1000, dynamic=dynamic)
    dt = time.perf_counter() - t0
    trees[dynamic] = tree
    nodes = count(tree)
    print(json.dumps({"config": "C3 CART", "dynamic": dynamic, "fact_rows": rows, "features": len(feats),
                      "thresholds": 20, "depth": 4, "nodes": nodes, "wall_s": dt, "ms_per_node": 1e3 * dt / nodes,
                      "aggregates_per_node": 3 + 3 * 20 * len(feats),
                      "root_split": [tree.get("feature"), tree.get("threshold")],
                      "plan": e.plan_info().get("fast_path")}), flush=True)


def shape(n):  # the splits and node sizes (means may differ in the last bits between the two plans)
    return (n["n"], n.get("feature"), n.get("threshold"), n.get("categories"),
            shape(n["left"]) if "left" in n else None, shape(n["right"]) if "right" in n else None)


assert shape(trees[True]) == shape(trees[False])
e.close()
