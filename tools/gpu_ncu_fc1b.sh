#!/bin/bash
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout -s KILL 600 $NCU --set full --import-source on --clock-control none -k regex:ztp_gemm_kernel -s 26 -c 1 \
  -o gpurun_out/gemm_fc1_fwd -f python tools/one_step.py > gpurun_out/ncu_fc1.log 2>&1
$NCU -i gpurun_out/gemm_fc1_fwd.ncu-rep --page details > gpurun_out/fc1_details.txt 2>&1
$NCU -i gpurun_out/gemm_fc1_fwd.ncu-rep --page source --csv --print-source sass > gpurun_out/fc1_sass.csv 2>&1
$NCU -i gpurun_out/gemm_fc1_fwd.ncu-rep --page source --csv > gpurun_out/fc1_src.csv 2>&1
tail -2 gpurun_out/ncu_fc1.log
