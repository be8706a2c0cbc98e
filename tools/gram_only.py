"""Standalone fact-only Gram (SURVEY §8(d) "(d) DMMA Gram"): the covariance batch of one relation
with 8 fp64 features (36 pair sums + 8 linear + count) at 10M and 100M rows — no dimensions, so
the scan is k_cov with no level structure.  Prints lmfao_run time, rows/s and the fraction of the
measured HBM copy bandwidth for 64 B/row.  usage: python tools/gram_only.py [rows ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1906_08687_b200 import lmfao  # noqa: E402

peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
for n in [int(x) for x in sys.argv[1:]] or [10_000_000, 100_000_000]:
    g = torch.Generator(device="cuda").manual_seed(0)
    cols = {f"x{j}": torch.randn(n, dtype=torch.float64, device="cuda", generator=g) for j in range(8)}
    feats = list(cols)
    e = lmfao.Engine()
    e.add_relation("F", cols)
    e.set_join_tree("F", [])
    e.prepare()
    e.add_query([], list(synth.covar_batch(feats).udafs))
    e.plan()
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    for _ in range(3):
        e.run(st.cuda_stream)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    a.record(st)
    for _ in range(reps):
        e.run(st.cuda_stream)
    b.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    gbs = 64.0 * n / (ms * 1e-3) / 1e9
    print(json.dumps({"rows": n, "features": 8, "run_ms": ms, "rows_per_s": n / (ms * 1e-3), "alg_gb_s": gbs,
                      "frac_hbm": gbs / peaks["hbm_gbs"], "plan": e.plan_info().get("fast_path")}), flush=True)
    e.close()
    del cols
    torch.cuda.empty_cache()
