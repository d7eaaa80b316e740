#!/bin/bash
# GPU: full bench line, ncu launch list of a short bench, ncu --set full of the decision kernels
# and of the 2^20 scan.  Outputs under gpurun_out/ (summarised into profiles/ by ncu_summary.py).
TAG=${1:-v6}
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -1 gpurun_out/bench_$TAG.json | cut -c1-400
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-sweep \
  > /dev/null 2> gpurun_out/launches_$TAG.err
DECISIONS=2 QOE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ -c 10 \
  -o gpurun_out/full_dec_$TAG -f python tools/profile_decision.py > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_qoe_scan -s 2 -c 1 \
  -o gpurun_out/full_scan1m_$TAG -f python tools/profile_scan.py > /dev/null 2>&1
ls -la gpurun_out/ | grep $TAG
