"""Per-source-line warp-stall samples (where warps spend their time) from `ncu --page source
--csv --print-source cuda,sass`: the SASS rows under each source line carry 'Warp Stall Sampling
(All Samples)' and the per-reason stall columns.  Usage: ncu_stall_lines.py file.csv [top]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1], encoding="latin1")))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, hdr = "", None
agg = defaultdict(float)
why = defaultdict(lambda: defaultdict(float))
text = {}
cur = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not r or r[0] == "Function Name" or hdr is None:
        continue
    if r[0]:  # a source line row
        cur = f"{fname}:{r[0]}"
        text[cur] = r[1].strip()[:90]
        continue
    # SASS row under cur
    try:
        s = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError:
        continue
    agg[cur] += s
    for j, h in enumerate(hdr):
        if h.startswith("stall_"):
            try:
                why[cur][h[6:]] += float(r[j] or 0)
            except ValueError:
                pass
tot = sum(agg.values())
print(f"total stall samples {tot:.0f}")
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    w = sorted(why[k].items(), key=lambda x: -x[1])[:3]
    print(f"{k:28s} {100 * v / tot:6.2f}%  {' '.join(f'{a}={100 * b / max(v, 1):.0f}%' for a, b in w)}  {text.get(k, '')}")
