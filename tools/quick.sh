#!/bin/bash
# GPU quick check: parity suite, long-request repro, short bench (stage breakdown + S1 QoE eval).
timeout 700 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
timeout 300 python tools/repro_long2.py 2>&1 | grep fails | tr '\n' ' '; echo
timeout 400 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/quick.json 2> gpurun_out/quick.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/quick.json").read().strip().splitlines()[-1])
r = d["roofline"]; q = d["qoe_eval"]
print("ms/decision", round(d["ms_per_step"], 4), {k: round(v * 1e3, 1) for k, v in r["stage_ms"].items()}, "us")
print("qoe 1M ms", round(q["ms_per_eval"], 4), "scan ms", round(q["scan_ms"], 4), "frac", round(q["roofline"]["frac"], 3))
PY
