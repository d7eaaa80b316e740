"""Group an ncu source-page CSV (SASS) into basic blocks by execution count; print the hottest."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ie = h.index("Instructions Executed"); isrc = h.index("Source"); ia = h.index("Address")
iss = h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    if len(r) <= ie or not r[ie].strip().isdigit():
        continue
    data.append((r[ia], r[isrc], int(r[ie]), int(r[iss] or 0)))
tot = sum(d[2] for d in data); ts = sum(d[3] for d in data) or 1
print("total warp instr", tot, "samples", ts)
blocks = []
for a, s, c, st in data:
    if blocks and blocks[-1][2] == c:
        blocks[-1][1].append(s); blocks[-1][3] += st
    else:
        blocks.append([a, [s], c, st])
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
full = len(sys.argv) > 3
for a, ss, c, st in sorted(blocks, key=lambda b: -b[2] * len(b[1]))[:n]:
    print(a, "count", c, "len", len(ss), f"{100 * c * len(ss) / tot:.1f}%", "stall%", f"{100 * st / ts:.1f}", "|",
          (" ; ".join(ss) if full else " ; ".join(x.split()[0] if x else "" for x in ss[:14])))
