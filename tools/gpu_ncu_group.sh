#!/bin/bash
# ncu --set full of the grouped O-projection dX+dW launch (3rd grouped launch of the 3rd step)
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
ZTP_GROUP=1 timeout -s KILL 600 $NCU --set full --import-source on --clock-control none -k regex:ztp_gemm_group_kernel -s 10 -c 1 \
  -o gpurun_out/group_o -f python tools/one_step.py > gpurun_out/ncu_group.log 2>&1
tail -2 gpurun_out/ncu_group.log
$NCU -i gpurun_out/group_o.ncu-rep --page details > gpurun_out/group_o_details.txt 2>&1
$NCU -i gpurun_out/group_o.ncu-rep --page raw --csv > gpurun_out/group_o_raw.csv 2>&1
