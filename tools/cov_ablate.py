"""Diagnostics for the k_cov scan: time lmfao_run on C2 with parts of the kernel
switched off (LMFAO_COV_ABLATE bitmask: 1 no gathers, 2 no record DMMA, 8 no H_L; results are
invalid in those modes; 16 pipeline only, 32 all blocks on the fast path, 64 no wait for the
gathers).  MODES=a,b,... picks the masks.
usage: LMFAO_NO_GRAPH=1 python tools/cov_ablate.py [fact_rows]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1906_08687_b200 import lmfao  # noqa: E402

kw = {"fact_rows": int(sys.argv[1])} if len(sys.argv) > 1 else {}
w = synth.config2(**kw)
e = lmfao.Engine()
lmfao.load(e, w.db, w.batch)
e.plan()
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
modes = [(12, int(m)) for m in os.environ["MODES"].split(",")] if "MODES" in os.environ else \
    [(12, 0), (12, 1), (12, 2), (12, 8), (12, 16), (12, 32), (12, 33), (12, 64), (12, 96), (12, 0)]
for wv, mode in modes:
    os.environ["LMFAO_COV_ABLATE"] = str(mode)
    for _ in range(3):
        e.run(st.cuda_stream)
    e.profile(True)
    for _ in range(20):
        e.run(st.cuda_stream)
    ms, n = e.profile_read()
    e.profile(False)
    print(json.dumps({"warps": wv, "ablate": mode, "scan_ms": ms / max(n, 1)}), flush=True)
