#!/bin/bash
# ncu --set full of the c0 TP=8 gamma=0.9 FC1 dX GEMM (17 computed, 119 all-pruned Zero tiles)
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
# launches per step: select, gather, 4 FWD GEMMs (+core, gather_rows), then BWD: FC2 dX is the 1st <1,...>, FC1 dX the 2nd
CFG=c0 TP=8 GAMMAS=0.9 timeout -s KILL 600 $NCU --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k regex:'gemm_kernel<.int.1, .int.2' -s 2 -c 1 -o gpurun_out/zero_fc1dx -f python tools/gamma_overhead.py > gpurun_out/ncu_zero.log 2>&1
$NCU -i gpurun_out/zero_fc1dx.ncu-rep --page details > gpurun_out/zero_fc1dx_details.txt 2>&1
$NCU -i gpurun_out/zero_fc1dx.ncu-rep --page source --csv > gpurun_out/zero_fc1dx_source.csv 2>&1
