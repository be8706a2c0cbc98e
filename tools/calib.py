"""Calibration runs of the Gram kernel on C2 (10M rows) with feature subsets:
NS=0 (fact + D3 only), NS=1 (fact + D2 + D3), NS=2 (all).  Prints kernel ms (CUDA events
around the scan kernel, lmfao_profile) per variant."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1906_08687_b200 import lmfao  # noqa: E402

w = synth.config2()
fx = [f"x{j}" for j in range(1, 9)]
d = lambda r: [f"d{r}_{j}" for j in range(1, 11)]
variants = {"NS0_fact+D3": fx + d(3), "NS1_fact+D2+D3": fx + d(2) + d(3), "NS2_all": fx + d(1) + d(2) + d(3),
            "NS0_D3only": d(3)}
torch.cuda.set_stream(torch.cuda.Stream())
for name, feats in variants.items():
    e = lmfao.Engine()
    lmfao.load(e, w.db, [synth.covar_batch(feats)])
    e.plan()
    sp = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        e.run(sp)
    torch.cuda.synchronize()
    e.profile(True)
    for _ in range(20):
        e.run(sp)
    ms, n = e.profile_read()
    print(f"{name:18s} {ms / n:8.3f} ms/launch  plan={e.plan_info()['fast_path']}", flush=True)
    e.close()
