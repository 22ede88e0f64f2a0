#!/bin/bash
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout -s KILL 200 python tools/gemm_bench.py --gammas 0,0.5 2>&1 | tee gpurun_out/gemm_bench.txt
GAMMA=0 timeout -s KILL 600 $NCU --set full --clock-control none --import-source on -k regex:ztp_gemm_kernel -s 3 -c 3 -o gpurun_out/gemm_full2 -f python tools/ncu_gemm.py > gpurun_out/ncu_full.log 2>&1
