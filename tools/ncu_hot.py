"""Hottest SASS instructions of an ncu --set full capture by warp-stall samples, with
the dominant stall reasons and the executed-instruction count per instruction.
usage: python tools/ncu_hot.py REP.ncu-rep [top=40] [context=0]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.split("\n")
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
h = rows[0]
idx = {k: i for i, k in enumerate(h)}
stall_cols = [c for c in h if c.startswith("stall_")]
recs = []
for r in rows[1:]:
    if len(r) < len(h):
        continue
    try:
        s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        ex = int(r[idx["Instructions Executed"]] or 0)
    except ValueError:
        continue
    st = sorted(((int(r[idx[c]] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
    recs.append((s, ex, r[idx["Address"]][-5:], r[idx["Source"]].strip(), st))
tot = sum(x[0] for x in recs)
print(f"total stall samples {tot}, instructions {len(recs)}")
for i, (s, ex, a, src, st) in enumerate(recs):
    recs[i] = (s, ex, a, src, st, i)
for s, ex, a, src, st, i in sorted(recs, reverse=True)[:top]:
    print(f"{100.0 * s / tot:5.1f}% {ex:>10} {a} {src[:60]:60s} " + " ".join(f"{n}:{v}" for v, n in st if v))
