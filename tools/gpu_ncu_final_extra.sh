#!/bin/bash
# ncu --set full of the c2 FC1 FWD (two-plane GeLU epilogue, the slowest GEMM per FLOP) and QKV dX, final kernels
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
CFG=c2 STEPS=0 timeout -s KILL 600 $NCU --set full --clock-control none --kernel-name-base demangled -k regex:'gemm_kernel<.int.0' -s 6 -c 1 -o gpurun_out/fc1_fwd_final -f python tools/one_step.py > /dev/null 2>&1
CFG=c2 STEPS=0 timeout -s KILL 600 $NCU --set full --clock-control none --kernel-name-base demangled -k regex:'gemm_kernel<.int.1' -s 7 -c 1 -o gpurun_out/qkv_dx_final -f python tools/one_step.py > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
