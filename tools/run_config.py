"""Load one config through the C-ABI and run it a few times (profiling driver).
usage: python tools/run_config.py [C2] [runs]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1906_08687_b200 import lmfao  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 3
kw = {}
if len(sys.argv) > 3:
    kw["fact_rows"] = int(sys.argv[3])
w = synth.CONFIGS[name](**kw)
e = lmfao.Engine()
q = lmfao.load(e, w.db, w.batch)
e.plan()
for _ in range(runs):
    e.run()
k, v, c = e.fetch(q[0])
print(name, "count", int(c[0]) if len(c) else None, e.plan_info().get("fast_path"))
