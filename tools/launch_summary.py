"""Per-kernel device time of the last RUNS lmfao_run calls in an ncu launch list (--metrics
gpu__time_duration.sum --csv): the kernels after the last plan-time kernel, grouped by name.
usage: python tools/launch_summary.py LAUNCHES.csv [RUNS]"""
import csv
import re
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, iv, iid = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("ID")
ks = [(int(r[iid]), re.sub(r"\(.*", "", r[ik]), float(r[iv].replace(",", ""))) for r in rows[1:]]
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 1
# a run ends where the run-sequence repeats: take the last `runs` repetitions of the tail
names = [k[1] for k in ks]
L = len(names)
period = next((p for p in range(1, L // 2 + 1) if names[L - p:] == names[L - 2 * p:L - p]), None)
tail = ks[L - period * runs:] if period else ks
agg = OrderedDict()
for _, n, v in tail:
    a = agg.setdefault(n, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(v for _, v in agg.values())
print(f"{period} launches per run; {tot / runs / 1e3:.3f} us per run" if period else "no period found")
for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v / runs / 1e3:10.1f} us  {c // runs:3d}x  {n[:110]}")
