#!/bin/bash
mkdir -p gpurun_out
for v in 1.0 1.2 1.4; do
  ZTP_AUX_WEIGHT=$v timeout -s KILL 300 python tools/graph_timeline.py > gpurun_out/auxw2_graph_$v.txt 2>&1
  ZTP_AUX_WEIGHT=$v timeout -s KILL 300 python tools/graph_timeline.py > gpurun_out/auxw2b_graph_$v.txt 2>&1
done
R=3 bash tools/gpu_ab2.sh ZTP_AUX_WEIGHT=1.0 ZTP_AUX_WEIGHT=1.2 ZTP_AUX_WEIGHT=1.4
for f in gpurun_out/auxw2*_graph_*; do echo "$f $(tail -1 $f)"; done
cat gpurun_out/ab2.txt
