#!/bin/bash
# ncu --set full of one GEMM variant from tools/epi_exp2.py (arg: case name)
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
CASE=${1:-fc1_fwd_gelu}
timeout -s KILL 600 $NCU --set full --import-source on --clock-control none -k regex:ztp_gemm_kernel -s 3 -c 1 \
  -o gpurun_out/$CASE -f python tools/epi_exp2.py 0 $CASE > gpurun_out/ncu_$CASE.log 2>&1
tail -2 gpurun_out/ncu_$CASE.log
