"""Attribute ncu per-instruction execution counts to CUDA source lines.

    python tools/sass_lines.py <report.ncu-rep> <kernel-regex> <object.o> <mangled-fn> [top]

Joins ncu's SASS source page (Instructions Executed per address) with
nvdisasm -g line info of the same function (offsets from the function start)."""
import collections
import csv
import io
import re
import subprocess
import sys
import tempfile
import os


def main():
    rep, kre, obj, fn = sys.argv[1:5]
    top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass", "-k", f"regex:{kre}"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia, isrc, iadr = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Address")
    iss = hdr.index("Warp Stall Sampling (All Samples)")
    cnt = []
    for r in rows[2:]:
        try:
            cnt.append((int(r[iadr], 16), int(r[ia]), r[isrc].strip(), int(r[iss] or 0)))
        except (ValueError, IndexError):
            pass
    base = cnt[0][0]
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    full = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
    start = full.index(f"//--------------------- .text.{fn} ")
    end = full.find("//--------------------- ", start + 10)
    sass = full[start:end if end > 0 else len(full)]
    line_of = {}
    cur = None
    for ln in sass.splitlines():
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
        if m and cur:
            line_of[int(m.group(1), 16)] = cur
    agg = collections.Counter()
    stl = collections.Counter()
    tot = tst = 0
    for adr, n, src, st in cnt:
        agg[line_of.get(adr - base, "?")] += n
        stl[line_of.get(adr - base, "?")] += st
        tot += n
        tst += st
    print("total instr", tot, "stall samples", tst)
    key = stl if os.environ.get("BY_STALL") else agg
    for k, v in key.most_common(top):
        print(f"{agg[k]:>10} {100 * agg[k] / tot:5.1f}%  stalls {stl[k]:>5} {100 * stl[k] / max(tst, 1):5.1f}%  {k}")


if __name__ == "__main__":
    main()
