"""Standalone view-build benchmark (kernel (b)): a many-to-many child D of
50M rows with 10 fp64 features and keys Zipf(1.1) over 1M values under a 1M-row root F;
batch COUNT + SUM(d_i) (the view of D has 11 slots).  Prints lmfao_run time; run under the
ncu launch list to isolate k_view_build.
usage: python tools/view_bench.py [child_rows] [keys]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1906_08687_b200 import lmfao  # noqa: E402

nd = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000_000
nk = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
rng = np.random.default_rng(0)
keys = np.arange(nk, dtype=np.int32)
D = {"k": keys[synth.zipf_ranks(rng, nk, 1.1, nd)].astype(np.int32)}
for j in range(10):
    D[f"d{j}"] = rng.standard_normal(nd)
F = {"k": rng.integers(0, nk, 1_000_000).astype(np.int32), "x": rng.standard_normal(1_000_000)}
db = synth.Database([synth.Relation("F", F), synth.Relation("D", D)], "F", [("F", "D")])
batch = [synth.Query([], [[synth.Product(1.0, ())]] + [[synth.Product(1.0, (synth.ident(f"d{j}"),))]
                                                       for j in range(10)])]
e = lmfao.Engine()
lmfao.load(e, db, batch)
e.plan()
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
for _ in range(2):
    e.run(st.cuda_stream)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(st)
for _ in range(5):
    e.run(st.cuda_stream)
b.record(st)
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 5
print(json.dumps({"child_rows": nd, "keys": nk, "slots": 11, "run_ms": ms,
                  "child_bytes": nd * 84, "plan": e.plan_info().get("fast_path")}), flush=True)
