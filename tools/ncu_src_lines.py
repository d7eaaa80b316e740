"""Per-source-line executed warp instructions from `ncu --page source --csv --print-source
cuda,sass` (the SASS rows under each source line carry the counts).  Usage: ncu_src_lines.py
file.csv [top] [source file for line text]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
srcs = {}
fname, cur = "", None
agg = defaultdict(int)
tot = 0
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1]
        continue
    if r and r[0] in ("Line No", "Function Name"):
        continue
    if r and r[0]:
        try:
            cur = (fname, int(r[0]))
        except ValueError:
            pass
        continue
    if len(r) > 7 and r[7] not in ("", "-"):
        v = int(r[7])
        agg[cur] += v
        tot += v
print("total warp instructions", tot)
for (f, l), v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    try:
        if f not in srcs:
            srcs[f] = open(f).read().splitlines()
        txt = srcs[f][l - 1].strip()[:90]
    except OSError:
        txt = ""
    print(f"{f.split('/')[-1]}:{l:<5d} {100 * v / tot:5.2f}%  {txt}")
