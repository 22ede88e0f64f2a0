#!/bin/bash
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
M="gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active,lts__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,smsp__inst_executed.sum,launch__grid_size,sm__cycles_active.avg"
ZTP_CONC=0 timeout -s KILL 300 $NCU --metrics $M --clock-control none -k regex:ztp_gemm_kernel -s 24 -c 12 --csv python tools/one_step.py > gpurun_out/ncu_dx_regular.csv 2>&1
