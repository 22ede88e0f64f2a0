#!/bin/bash
# per-kernel launch list of one c0 TP=8 rank's step at gamma 0 / 0.5 / 0.9 (what a heavily resized straggler pays)
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
CFG=c0 TP=8 GAMMAS=0,0.5,0.9 timeout -s KILL 600 $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:ztp --csv \
  --log-file gpurun_out/gov_c0.csv python tools/gamma_overhead.py > gpurun_out/gov_c0.log 2>&1
CFG=c0 TP=8 GAMMAS=0,0.5,0.9 python tools/gamma_overhead.py --parse gpurun_out/gov_c0.csv gpurun_out/gov_c0.json > gpurun_out/gov_c0.txt 2>&1
cat gpurun_out/gov_c0.txt
