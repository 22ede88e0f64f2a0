#!/bin/bash
mkdir -p gpurun_out
for d in 0 1 2; do
  echo "dbg=$d"; ZTP_DEBUG_EPI=$d timeout -s KILL 200 python tools/gemm_bench.py --shapes "1024,4096,8192;4096,1024,8192" --gammas 0,0.5
done 2>&1 | tee gpurun_out/exp.txt
