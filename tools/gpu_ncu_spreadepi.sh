#!/bin/bash
# ncu --set full of the c4 FC1 dW GEMM (output-pruned, unsplit) with the column spread in its epilogue
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
CFG=c4 STEPS=0 timeout -s KILL 900 $NCU --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:'gemm_kernel<.int.2' -s 5 -c 1 -o gpurun_out/spreadepi_c4 -f python tools/one_step.py > gpurun_out/ncu_spreadepi.log 2>&1
$NCU -i gpurun_out/spreadepi_c4.ncu-rep --page details > gpurun_out/spreadepi_c4_details.txt 2>&1
$NCU -i gpurun_out/spreadepi_c4.ncu-rep --page source --csv > gpurun_out/spreadepi_c4_source.csv 2>&1
