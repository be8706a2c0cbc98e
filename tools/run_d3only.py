import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_1906_08687_b200 import lmfao
w = synth.config2()
e = lmfao.Engine()
lmfao.load(e, w.db, [synth.covar_batch([f"d3_{j}" for j in range(1, 11)])])
e.plan()
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    e.run()
print(e.fetch(0)[2])
