#!/bin/bash
# full ncu sections of the column-spread kernels: expand_cols (c4 dW1) and dw_reduce<2,1> (c2 FC1 dW)
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
CFG=c4 timeout -s KILL 600 $NCU --set full --import-source on --clock-control none -k regex:ztp_expand_cols -s 2 -c 1 -o gpurun_out/expand_c4 -f python tools/one_step.py > gpurun_out/ncu_expand.log 2>&1
CFG=c2 timeout -s KILL 600 $NCU --set full --import-source on --clock-control none -k regex:ztp_dw_reduce -s 2 -c 1 -o gpurun_out/dwred_c2 -f python tools/one_step.py > gpurun_out/ncu_dwred.log 2>&1
for f in expand_c4 dwred_c2; do $NCU -i gpurun_out/$f.ncu-rep --page details > gpurun_out/${f}_details.txt 2>&1; $NCU -i gpurun_out/$f.ncu-rep --page source --csv > gpurun_out/${f}_source.csv 2>&1; done
