"""Per-kernel device time of the last N launches of an ncu launch list (--metrics
gpu__time_duration.sum --csv), grouped by kernel name.
usage: python tools/last_run_kernels.py LAUNCHES.csv N [SKIP]   (SKIP: ignore the last SKIP launches,
e.g. the compaction of a fetch after the last run)"""
import csv
import re
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ik, iv, iid = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
ks = [(int(r[iid]), re.sub(r"\(.*", "", r[ik]), float(r[iv].replace(",", ""))) for r in rows[1:]]
agg = OrderedDict()
skip = int(sys.argv[3]) if len(sys.argv) > 3 else 0
sel = ks[len(ks) - skip - int(sys.argv[2]):len(ks) - skip]
for _, n, v in sel:
    a = agg.setdefault(n, [0, 0.0])
    a[0] += 1
    a[1] += v
print(f"{sum(v for _, v in agg.values()) / 1e3:.1f} us in the last {sys.argv[2]} launches")
for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v / 1e3:10.1f} us {c:4d}x  {n[:100]}")
