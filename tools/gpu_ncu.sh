#!/bin/bash
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
ACT=gelu GAMMA=0.5 timeout -s KILL 600 $NCU --set full --clock-control none -k regex:ztp_gemm_kernel -s 3 -c 2 -o gpurun_out/gelu512 -f python tools/ncu_gemm.py > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
