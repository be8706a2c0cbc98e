"""C3 with a tree-node path condition on every aggregate: lmfao_run
on the rt.cu path (filter + conditioned pass + unconditioned multiplicity pass) and, with
--generic, on the interpreted path.  usage: python tools/time_rt_path.py [fact_rows] [--generic] [--ct]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1906_08687_b200 import lmfao  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 10_000_000
w = synth.config3(fact_rows=rows)
path = (synth.Factor(synth.F_GE, "x1", -0.5), synth.Factor(synth.F_LE, "d2_1", 0.25),
        synth.Factor(synth.F_GT, "d3_1", -1.0))
if "--ct" in sys.argv:  # a classification node: CT(c1; α), CT(c1; α·1[A <= t]) per feature A, CT(α)
    feats = w.meta["features"]
    ts = synth.thresholds_c3()
    batch = [synth.Query(["c1"], [[synth.Product(1.0, path)]])]
    batch += [synth.Query(["c1"], [[synth.Product(1.0, path + (synth.Factor(synth.F_LE, a, t),))] for t in ts])
              for a in feats]
    batch.append(synth.Query([], [[synth.Product(1.0, path)]]))
else:
    batch = [synth.Query(q.groupby, [[synth.Product(p.coeff, path + tuple(p.factors)) for p in u] for u in q.udafs])
             for q in w.batch]
if "--generic" in sys.argv:
    os.environ["LMFAO_GENERIC_ONLY"] = "1"
torch.cuda.set_stream(torch.cuda.Stream())
cols = {r.name: {c: torch.from_numpy(v).cuda() for c, v in r.cols.items()} for r in w.db.relations}
e = lmfao.Engine()
q = lmfao.load(e, w.db, batch, columns=cols)
e.plan()
sp = torch.cuda.current_stream().cuda_stream
e.run(sp)
e.run(sp)
torch.cuda.synchronize()
s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 3 if "--generic" in sys.argv else 20
s.record()
for _ in range(n):
    e.run(sp)
t.record()
torch.cuda.synchronize()
print(json.dumps({"config": "C3+path3" + ("+ct(c1)" if "--ct" in sys.argv else ""), "fact_rows": rows, "aggregates": synth.n_aggregates(batch),
                  "run_ms": s.elapsed_time(t) / n, "plan": e.plan_info().get("fast_path")}))
