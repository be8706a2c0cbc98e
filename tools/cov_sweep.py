"""Diagnostics for the k_cov scan on C2: re-plan under plan-time knobs (PLAN: ';'-separated sets of
'VAR=v,VAR=v' environment assignments, e.g. LMFAO_COV_IB / LMFAO_COV_TB / LMFAO_COV_TAIL, the work-item
sizes) and time the scan under run-time ablations (LMFAO_COV_ABLATE, results invalid: 1 no gathers,
8 no H_L, 16 pipeline only, 32 every block on the fast path).
usage: python tools/cov_sweep.py [PLAN=..] [ABLATE=a1,a2,..] [ROWS=n]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1906_08687_b200 import lmfao  # noqa: E402

opt = dict(a.split("=", 1) for a in sys.argv[1:])
plans = [dict(kv.split("=", 1) for kv in p.split(",") if kv) for p in opt.get("PLAN", "").split(";")]
ablates = [int(x) for x in opt.get("ABLATE", "0").split(",")]
kw = {"fact_rows": int(opt["ROWS"])} if "ROWS" in opt else {}
w = synth.config2(**kw)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
for plan in plans:
    os.environ.update(plan)
    e = lmfao.Engine()
    lmfao.load(e, w.db, w.batch)
    e.plan()
    for ab in ablates:
        os.environ["LMFAO_COV_ABLATE"] = str(ab)
        for _ in range(3):
            e.run(st.cuda_stream)
        e.profile(True)
        for _ in range(30):
            e.run(st.cuda_stream)
        ms, n = e.profile_read()
        e.profile(False)
        print(json.dumps({"plan": plan, "ablate": ab, "scan_ms": round(ms / max(n, 1), 4),
                          "info": e.plan_info().get("fast_path")}), flush=True)
    os.environ["LMFAO_COV_ABLATE"] = "0"
    for k in plan:
        del os.environ[k]
    e.close()
