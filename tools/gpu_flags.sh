#!/bin/bash
# tile-completion flags between consecutive GEMMs: parity with the flags on, timelines and bench A/B
mkdir -p gpurun_out
ZTP_FLAGS=1 timeout -s KILL 900 python -m pytest tests/test_gpu_runtime.py tests/test_gpu_layer.py tests/test_gpu_kernels.py -x -q -m gpu 2>&1 | tail -15 > gpurun_out/flags_tests.txt
cat gpurun_out/flags_tests.txt | tail -3
for v in 0 1; do
  ZTP_FLAGS=$v timeout -s KILL 300 python tools/cta_timeline.py > gpurun_out/flags_cta_$v.txt 2>&1
  ZTP_FLAGS=$v timeout -s KILL 300 python tools/graph_timeline.py > gpurun_out/flags_graph_$v.txt 2>&1
  echo "flags=$v $(tail -1 gpurun_out/flags_graph_$v.txt)"
done
R=3 bash tools/gpu_ab2.sh ZTP_FLAGS=0 ZTP_FLAGS=1
cat gpurun_out/ab2.txt
