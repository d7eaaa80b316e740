"""Summarise ncu reports / launch lists into profiles/*.md (run on the CPU box)."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("smsp__inst_executed.sum", "warp instr"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def rep_summary(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out = ["| kernel | " + " | ".join(k[1] for k in KEYS) + " | top stalls (per issue) |",
           "|---" * (len(KEYS) + 2) + "|"]
    st = [c for c in h if c.startswith("smsp__average_warps_issue_stalled_") and c.endswith("_per_issue_active.ratio")]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("andes::", "")
        vals = []
        for k, _ in KEYS:
            if k in h:
                v = r[h.index(k)]
                u = units[h.index(k)]
                vals.append(f"{v} {u}".strip())
            else:
                vals.append("-")
        s = sorted([(float(r[h.index(c)] or 0), c.replace("smsp__average_warps_issue_stalled_", "").replace(
            "_per_issue_active.ratio", "")) for c in st], reverse=True)[:4]
        out.append(f"| {name} | " + " | ".join(vals) + " | " + ", ".join(f"{n} {v:.2f}" for v, n in s) + " |")
    return "\n".join(out)


def launches_summary(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("andes::", "").replace("void ", "")
        v = float(r[vi].replace(",", ""))
        if r[ui] == "usecond":
            v *= 1000
        elif r[ui] == "msecond":
            v *= 1e6
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for k, a in agg.items() if "andes" in k or k.startswith("k_"))
    out = ["| kernel | launches | total ns | mean ns | share of andes time |", "|---|---|---|---|---|"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        mine = k.startswith("k_")
        share = f"{t / tot:.3f}" if mine and tot else "-"
        out.append(f"| {k} | {c} | {t:.0f} | {t / c:.0f} | {share} |")
    return "\n".join(out)


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(rep_summary(path) if kind == "rep" else launches_summary(path))
