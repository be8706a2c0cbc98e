"""Key numbers of an ncu --set full capture: duration, IPC, dram bytes, FP64 pipe, stall mix, SM balance.
usage: python tools/ncu_summary.py REP.ncu-rep [--json out.json]"""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h, units, v = r[0], r[1], r[2]
d = dict(zip(h, v))
u = dict(zip(h, units))


def f(k):
    try:
        return float(d[k].replace(",", ""))
    except Exception:
        return None


keys = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg", "sm__cycles_active.avg", "sm__cycles_active.min",
        "sm__cycles_active.max", "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "lts__t_sector_hit_rate.pct", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
res = {k: (f(k), u.get(k)) for k in keys if k in d}
for k, (val, unit) in res.items():
    print(f"{k:70s} {val} {unit}")
st = [(k, f(k)) for k in h if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")]
tot = sum(x for _, x in st if x)
for k, x in sorted(st, key=lambda z: -(z[1] or 0))[:8]:
    print(f"  stall {100 * x / tot:5.1f}%  {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}")
atom = [k for k in h if k.endswith(".sum") and not k.startswith("sys") and "aperture" not in k and "lookup" not in k
        and any(t in k for t in ("op_atom", "op_red", "shared_atom", "global_red", "global_atom"))]
if atom:
    print("-- atomics / reductions")
    for k in sorted(atom):
        if f(k):
            print(f"{k:80s} {f(k):.0f}")
if "--json" in sys.argv:
    json.dump({k: val for k, (val, unit) in res.items()}, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
