#!/bin/bash
# ncu --set full (source view) of the c2 FC1 FWD GEMM (two-plane GeLU / GeLU' epilogue), 3rd FWD GEMM of step 2
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
CFG=c2 STEPS=0 timeout -s KILL 900 $NCU --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:'gemm_kernel<.int.0' -s 6 -c 1 -o gpurun_out/fc1fwd_c2 -f python tools/one_step.py > gpurun_out/ncu_fc1fwd.log 2>&1
$NCU -i gpurun_out/fc1fwd_c2.ncu-rep --page details > gpurun_out/fc1fwd_c2_details.txt 2>&1
$NCU -i gpurun_out/fc1fwd_c2.ncu-rep --page source --csv > gpurun_out/fc1fwd_c2_source.csv 2>&1
