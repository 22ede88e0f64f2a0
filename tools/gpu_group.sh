#!/bin/bash
# grouped dX + dW launch: never (0) / always (1) / where it pays (2, default): parity + timeline
mkdir -p gpurun_out
rm -f gpurun_out/group_tl.txt
ZTP_GROUP=1 timeout -s KILL 600 python -m pytest tests/test_gpu_layer.py -x -q 2>&1 | tail -5 > gpurun_out/group_tests.txt
for g in 0 2 0 2; do
  echo "== ZTP_GROUP=$g" >> gpurun_out/group_tl.txt
  ZTP_GROUP=$g timeout -s KILL 300 python tools/graph_timeline.py >> gpurun_out/group_tl.txt 2>&1
done
