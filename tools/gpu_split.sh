#!/bin/bash
# experiment: a fixed dX / dW SM split for every linear (ZTP_DX_PAIRS) vs the work-proportional default
mkdir -p gpurun_out
for px in 0 30 37 44 0; do
  echo "== ZTP_DX_PAIRS=$px" >> gpurun_out/split.txt
  ZTP_DX_PAIRS=$px timeout -s KILL 300 python tools/graph_timeline.py >> gpurun_out/split.txt 2>&1
done
