"""Per-opcode and per-source-line execution counts of one kernel in an ncu report (dev tool).

    python tools/sass_ops.py rep.ncu-rep kernel-regex object.o mangled-fn [units] [OPS...]
units: divide counts by this (e.g. tiles per launch)."""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, kre, obj, fn = sys.argv[1:5]
units = float(sys.argv[5]) if len(sys.argv) > 5 else 1.0
ops = sys.argv[6:] or ["LOP3", "PRMT", "ISETP", "SEL", "IADD3", "VIADD", "HSET2", "HMNMX2", "VHMNMX", "SHF", "LEA"]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass", "-k", f"regex:{kre}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1] if "Source" not in rows[0] else rows[0]
st = 2 if hdr is rows[1] else 1
ia, isrc, iadr = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Address")
cnt = []
for r in rows[st:]:
    try:
        cnt.append((int(r[iadr], 16), int(r[ia]), r[isrc].strip()))
    except (ValueError, IndexError):
        pass
base = cnt[0][0]
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
full = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
s = full.index(f"//--------------------- .text.{fn} ")
e = full.find("//--------------------- ", s + 10)
line_of, cur = {}, None
for ln in full[s:e if e > 0 else len(full)].splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
tot = collections.Counter()
for a, n, src in cnt:
    o = src.split()
    if o:
        tot[(o[1] if o[0].startswith("@") else o[0]).split(".")[0]] += n
print("total", round(sum(tot.values()) / units, 1), [(k, round(v / units, 1)) for k, v in tot.most_common(20)])
for opn in ops:
    agg = collections.Counter()
    for a, n, src in cnt:
        o = src.split()
        if o and (o[1] if o[0].startswith("@") else o[0]).startswith(opn):
            agg[line_of.get(a - base, "?")] += n
    print(opn, [(k, round(v / units, 1)) for k, v in agg.most_common(8)])
