#!/bin/bash
# A/B of env toggles on the decision latency: bash tools/ab.sh "ENV=1" "ENV2=0" ...
for cfg in "" "$@"; do
  env $cfg timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-sweep --no-sharded > gpurun_out/ab.json 2> gpurun_out/ab.err
  python - "$cfg" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1]); r = d["roofline"]
print(f"[{(sys.argv[1] or 'default')[-40:]}] ms/decision", round(d["ms_per_step"], 4), {k: round(v * 1e3, 1) for k, v in r["stage_ms"].items()},
      {k: round(v["ms_per_decision"] * 1e3, 1) for k, v in d["objectives"].items()}, "scan1M", round(d["qoe_eval"]["scan_ms"], 4), "clk", d.get("clocks", {}).get("sm_mhz"))
PY
done
