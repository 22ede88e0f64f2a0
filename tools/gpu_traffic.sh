#!/bin/bash
# DRAM bytes per GEMM launch of one layer step (3rd step, 12 launches) per config at TP = 1, gamma = 0.5
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
for c in c2 c3 c4 c5; do
  CFG=$c timeout -s KILL 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:ztp_gemm_kernel -s 24 -c 12 --csv python tools/one_step.py > gpurun_out/traffic_$c.csv 2>&1
done
