"""Wall-clock phases of the end-to-end path (bench.py's e2e) on C2: add_relation from
pinned host memory, prepare (remap + sort), add_query + plan, run, fetch.
usage: python tools/e2e_phases.py [--keep]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1906_08687_b200 import lmfao  # noqa: E402

w = synth.config2()
keep = None
if "--keep" in sys.argv:  # like bench.py: a first engine with the same data stays alive
    keep = lmfao.Engine()
    lmfao.load(keep, w.db, w.batch)
    keep.plan()
    keep.run()
    torch.cuda.synchronize()
pinned = {r.name: {c: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for c, v in r.cols.items()}
          for r in w.db.relations}
for it in range(3):
    t = [time.perf_counter()]
    e = lmfao.Engine()
    for r in w.db.relations:
        e.add_relation(r.name, pinned[r.name])
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    e.set_join_tree(w.db.root, list(w.db.edges))
    e.prepare()
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    q = [e.add_query(list(qq.groupby), list(qq.udafs)) for qq in w.batch]
    e.plan()
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    e.run()
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    e.fetch(q[0])
    t.append(time.perf_counter())
    e.close()
    d = np.diff(t) * 1e3
    print(f"iter {it}: add_relation {d[0]:.1f} ms, prepare {d[1]:.1f} ms, plan {d[2]:.1f} ms, run {d[3]:.2f} ms, "
          f"fetch {d[4]:.2f} ms, total {sum(d):.1f} ms", flush=True)
