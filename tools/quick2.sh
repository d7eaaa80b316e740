#!/bin/bash
# GPU check: decision trace, parity + shard suites, short bench summary (stages, objectives, 1M scan)
python tools/trace_decision.py 2>&1 | grep -v tile
timeout 700 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -x -q 2>&1 | tail -2
timeout 400 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/quick.json 2> gpurun_out/quick.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/quick.json").read().strip().splitlines()[-1]); r = d["roofline"]; q = d["qoe_eval"]
print("ms/decision", round(d["ms_per_step"], 4), {k: round(v * 1e3, 1) for k, v in r["stage_ms"].items()},
      {k: round(v["ms_per_decision"] * 1e3, 1) for k, v in d["objectives"].items()})
print("qoe 1M ms", round(q["ms_per_eval"], 4), "scan", round(q["scan_ms"], 4), "frac", round(q["roofline"]["frac"], 3),
      "sharded", {k: v for k, v in (d.get("sharded") or {}).items() if "ms" in k})
PY
