#!/bin/bash
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout -s KILL 600 $NCU --set full --import-source on --clock-control none -k regex:ztp_gemm_kernel -s 26 -c 1 \
  -o gpurun_out/gemm_fc1_fwd -f python tools/one_step.py > gpurun_out/ncu_fc1.log 2>&1
tail -2 gpurun_out/ncu_fc1.log
