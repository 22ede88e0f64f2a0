#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -x -q -m gpu 2>&1 | tail -3 | tee gpurun_out/expand_tests.txt
NCU=/usr/local/cuda/bin/ncu
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum"
for c in c4 c5; do
  CFG=$c timeout -s KILL 600 $NCU --metrics $M --clock-control none -k regex:'ztp_(expand)' --csv python tools/one_step.py > gpurun_out/expand_$c.csv 2>&1
  python tools/summarize_ncu.py gpurun_out/expand_$c.csv --last 4 > gpurun_out/expand_$c.txt 2>&1
  cat gpurun_out/expand_$c.txt
done
CONFIGS="c4 c5" bash tools/gpu_configs.sh
