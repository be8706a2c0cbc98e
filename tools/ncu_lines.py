"""Attribute an ncu --set full capture to CUDA source lines (uses the SASS page and
nvdisasm -g line info of the compiled object).
usage: python tools/ncu_lines.py REP.ncu-rep OBJ.o MANGLED_KERNEL [groups]"""
import csv
import io
import re
import subprocess
import sys
import tempfile
from collections import Counter, defaultdict

import os
rep, obj, kern = sys.argv[1], os.path.abspath(sys.argv[2]), sys.argv[3]
units = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", obj], cwd=d, capture_output=True)
import glob
sass = []
for cub in glob.glob(d + "/*.cubin"):  # the cubin holding the kernel (a .so carries one per source file)
    sass = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout.split("\n")
    if any(f".text.{kern}:" in l for l in sass):
        break
start = next(i for i, l in enumerate(sass) if f".text.{kern}:" in l)
cur, a2l = None, {}
for l in sass[start + 1:]:
    if l.startswith(".text.") or (l.strip().startswith(".section") and a2l):
        break
    mm = re.search(r"line (\d+)", l)
    if mm and "##" in l:
        cur = int(mm.group(1))
        continue
    m2 = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", l)
    if m2:
        a2l[int(m2.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
ix = hdr.index("Instructions Executed")
samp = hdr.index("Warp Stall Sampling (All Samples)")
base = int(data[0][0], 16)
agg, sm, ops = defaultdict(float), defaultdict(int), Counter()
for r in data:
    ln = a2l.get(int(r[0], 16) - base)
    agg[ln] += int(r[ix] or 0)
    sm[ln] += int(r[samp] or 0)
    op = r[1].split()
    if op:
        o = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
        ops[o.split(".")[0]] += int(r[ix] or 0)
tot = sum(agg.values())
src_file = None
for l in sass:
    mm = re.search(r'File "([^"]+)"', l)
    if mm and kern[:10]:
        src_file = mm.group(1)
        break
src = open(src_file).read().split("\n") if src_file else []
print(f"total {tot:.0f} warp-instr, {tot / units:.1f} per unit")
for ln, n in sorted(agg.items(), key=lambda x: -x[1])[:int(os.environ.get("TOP", "35"))]:
    s = src[ln - 1].strip()[:95] if ln and ln <= len(src) else "?"
    print(f"{n / units:7.1f}  stall {sm[ln]:6d}  L{ln}  {s}")
print("top opcodes:", ", ".join(f"{o} {n / units:.1f}" for o, n in ops.most_common(12)))
