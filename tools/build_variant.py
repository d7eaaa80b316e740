"""Build a variant of libandes.so with extra -D flags (A/B timing via ANDES_LIB_PATH).
usage: python tools/build_variant.py OUT.so [-DNAME[=V] ...]"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2404_16283_b200"))
import build as B  # noqa: E402

out, defs = sys.argv[1], sys.argv[2:]
cmd = ["nvcc", *[f for f in B.NVCC_FLAGS if f != "-v" and f != "-Xptxas"], *defs, "-o", out,
       *[os.path.join(B.CSRC, s) for s in B.SOURCES]]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.stderr.write(r.stdout + r.stderr)
    sys.exit(1)
print(out)
