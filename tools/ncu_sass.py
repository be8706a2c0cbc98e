"""Hot SASS of an ncu --set full capture in address order: instructions executed at least MIN
times (default: once per unit), with their source line (nvdisasm -g of the object).
usage: python tools/ncu_sass.py REP.ncu-rep OBJ.o MANGLED_KERNEL UNITS [MINFRAC]"""
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile

rep, obj, kern, units = sys.argv[1], os.path.abspath(sys.argv[2]), sys.argv[3], float(sys.argv[4])
minfrac = float(sys.argv[5]) if len(sys.argv) > 5 else 0.9
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", obj], cwd=d, capture_output=True)
sass = []
for cub in glob.glob(d + "/*.cubin"):
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
hdr, data = rows[1], rows[2:]
ix = hdr.index("Instructions Executed")
base = int(data[0][0], 16)
for r in data:
    n = int(r[ix] or 0)
    if n >= minfrac * units:
        a = int(r[0], 16) - base
        print(f"{a:6x} L{a2l.get(a)!s:5s} {n / units:6.2f}  {r[1]}")
