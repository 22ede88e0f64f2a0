#!/bin/bash
# dX/dW SM partition: weight of a GeLU'-epilogue dX (FC2 BWD), graph timelines + interleaved bench
mkdir -p gpurun_out
for v in 1.0 1.4 1.7; do
  ZTP_AUX_WEIGHT=$v timeout -s KILL 300 python tools/graph_timeline.py > gpurun_out/auxw_graph_$v.txt 2>&1
done
R=4 bash tools/gpu_ab2.sh "ZTP_AUX_WEIGHT=1.0 ZTP_A_EARLY=0" "ZTP_AUX_WEIGHT=1.0" "ZTP_AUX_WEIGHT=1.4" "ZTP_AUX_WEIGHT=1.7"
cat gpurun_out/ab2.txt
