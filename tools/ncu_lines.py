"""Per-source-line instruction counts and stall samples from `ncu --page source --csv
--print-source cuda,sass` output (run on the CPU box). Usage: ncu_lines.py file.csv [top]"""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
agg = defaultdict(lambda: [0.0, 0.0, ""])
fname = ""
hdr = None
tot_i = tot_s = 0.0
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) // 2:
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    ie = hdr.index("Instructions Executed")
    ss = hdr.index("Warp Stall Sampling (All Samples)")
    try:
        i = float(r[ie] or 0)
        s = float(r[ss] or 0)
    except ValueError:
        continue
    a = agg[(fname, ln)]
    a[0] += i
    a[1] += s
    a[2] = r[1][:90]
    tot_i += i
    tot_s += s
print(f"total instr {tot_i:.3e}  samples {tot_s:.0f}")
for (f, ln), (i, s, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{f}:{ln:<5} instr {i / tot_i * 100:5.1f}%  stall {s / max(tot_s, 1) * 100:5.1f}%  {src.strip()}")
