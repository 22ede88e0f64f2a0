#!/bin/bash
# tests + per-kernel gamma overhead launch lists + recovery simulation + bench
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout -s KILL 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/gpu_tests.txt
for c in "c4 8" "c2 4"; do set -- $c
  CFG=$1 TP=$2 timeout -s KILL 400 $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:ztp --csv \
    --log-file gpurun_out/gov_$1_$2.csv python tools/gamma_overhead.py > gpurun_out/gov_$1_$2.log 2>&1
  CFG=$1 TP=$2 python tools/gamma_overhead.py --parse gpurun_out/gov_$1_$2.csv gpurun_out/gov_$1_$2.json > gpurun_out/gov_$1_$2.txt 2>&1
done
timeout -s KILL 900 python tools/recovery_sim.py > gpurun_out/recovery_sim.txt 2>&1
timeout -s KILL 400 python bench.py 2>&1 | tail -1 > gpurun_out/bench.txt
cat gpurun_out/gpu_tests.txt; grep -h "^gamma" gpurun_out/gov_*.txt; cat gpurun_out/bench.txt | cut -c1-400
