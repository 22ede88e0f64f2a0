#!/bin/bash
# contiguous-run fast path in the column-spread / split-K dW reduces: parity, configs, non-GEMM launch times
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -2 | tee gpurun_out/runs_tests.txt
CONFIGS="c2 c4 c5" bash tools/gpu_configs.sh > /dev/null 2>&1; cut -c1-175 gpurun_out/configs.txt
NCU=/usr/local/cuda/bin/ncu
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum"
for c in c2 c4; do
  CFG=$c timeout -s KILL 600 $NCU --metrics $M --clock-control none -k regex:'ztp_(dw_reduce|splitk|expand)' --csv python tools/one_step.py > gpurun_out/runs_$c.csv 2>&1
  python tools/summarize_ncu.py gpurun_out/runs_$c.csv 2>&1 | tail -4
done
