"""Time lmfao_run on full-size configs (device-resident inputs, CUDA events).
usage: python tools/time_configs.py C3 C4 ...   (prints one JSON line per config)"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1906_08687_b200 import lmfao  # noqa: E402

for name in sys.argv[1:] or ["C1", "C3", "C4"]:
    kw = {}
    if ":" in name:
        name, rows = name.split(":")
        kw["fact_rows"] = int(rows)
    t0 = time.perf_counter()
    w = synth.CONFIGS[name](**kw)
    tg = time.perf_counter() - t0
    e = lmfao.Engine()
    t0 = time.perf_counter()
    q = lmfao.load(e, w.db, w.batch)
    e.plan()
    torch.cuda.synchronize()
    tl = time.perf_counter() - t0
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    for _ in range(2):
        e.run(stream.cuda_stream)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    a.record(stream)
    for _ in range(reps):
        e.run(stream.cuda_stream)
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    t0 = time.perf_counter()
    shapes = [e.result_shape(i)[0] for i in q]
    tf = time.perf_counter() - t0
    n = w.db.rel(w.db.root).nrows
    print(json.dumps({"config": name, "fact_rows": n, "run_ms": ms, "rows_per_s": n / ms * 1e3, "gen_s": tg,
                      "load_plan_s": tl, "compact_s": tf, "groups": sum(shapes), "plan": e.plan_info().get("fast_path"),
                      "launches": e.plan_info().get("launches_last_run")}), flush=True)
    e.close()
    del w
