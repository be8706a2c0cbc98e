"""C5 run time under LMFAO_CUBE_ABLATE variants of the cube kernel (cube.cu): 0 full,
1 no flush (scans + memsets only), 2 counts only, 4 no flush at levels >= 2.
usage: python tools/cube_ablate.py [fact_rows]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1906_08687_b200 import lmfao  # noqa: E402

kw = {"fact_rows": int(sys.argv[1])} if len(sys.argv) > 1 else {}
w = synth.config5(**kw)
torch.cuda.set_stream(torch.cuda.Stream())  # a real stream: run(0) would mean the ctx stream
cols = {r.name: {c: torch.from_numpy(v).cuda() for c, v in r.cols.items()} for r in w.db.relations}
for ab in ["0", "1", "2", "4", "nocube"]:
    os.environ["LMFAO_CUBE_ABLATE"] = ab if ab != "nocube" else "0"
    os.environ["LMFAO_NO_CUBE"] = "1" if ab == "nocube" else "0"
    e = lmfao.Engine()
    q = lmfao.load(e, w.db, w.batch, columns=cols)
    e.plan()
    sp = torch.cuda.current_stream().cuda_stream
    e.run(sp)
    e.run(sp)
    torch.cuda.synchronize()
    s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(3):
        e.run(sp)
    t.record()
    torch.cuda.synchronize()
    print(json.dumps({"ablate": ab, "run_ms": s.elapsed_time(t) / 3, "plan": e.plan_info().get("fast_path", {}).get("kind")}),
          flush=True)
    e.close()
