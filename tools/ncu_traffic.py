"""Write profiles/ncu_traffic.json: DRAM bytes per launch (dram__bytes_read.sum +
dram__bytes_write.sum) of k_qoe_scan in the committed ncu --set full captures (CPU box).
Usage: ncu_traffic.py <decision .ncu-rep> <2^20 scan .ncu-rep> <source note>"""
import csv
import io
import json
import os
import subprocess
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def scan_bytes(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        if "k_qoe_scan" not in r[h.index("Kernel Name")]:
            continue
        tot = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tot += float(r[h.index(k)]) * UNIT[u[h.index(k)]]
        out.append(tot)
    return out


dec, big, note = sys.argv[1], sys.argv[2], sys.argv[3]
d = scan_bytes(dec)
b = scan_bytes(big)
res = {"k_qoe_scan_config3": round(sum(d) / len(d)), "k_qoe_scan_2p20": round(sum(b) / len(b)),
       "unit": "bytes per launch", "source": note}
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
json.dump(res, open(os.path.join(root, "profiles", "ncu_traffic.json"), "w"), indent=1)
print(res)
