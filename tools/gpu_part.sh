#!/bin/bash
# dX/dW partition model A/B (interleaved bench rounds) + graph timelines
mkdir -p gpurun_out
for v in "ZTP_AUX_WEIGHT=1.4" "ZTP_AUX_WEIGHT=1.4 ZTP_PART=1" "ZTP_AUX_WEIGHT=1.7 ZTP_PART=1"; do
  tag=$(echo $v | tr ' =' '_-')
  env $v timeout -s KILL 300 python tools/graph_timeline.py > gpurun_out/part_graph_$tag.txt 2>&1
done
R=3 bash tools/gpu_ab2.sh "ZTP_AUX_WEIGHT=1.4" "ZTP_AUX_WEIGHT=1.0 ZTP_PART=1" "ZTP_AUX_WEIGHT=1.4 ZTP_PART=1" "ZTP_AUX_WEIGHT=1.7 ZTP_PART=1" "ZTP_AUX_WEIGHT=1.4 ZTP_PART=1 ZTP_DW_SHARE=1.0"
cat gpurun_out/ab2.txt
