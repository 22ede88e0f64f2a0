#!/bin/bash
# ncu of the non-GEMM kernels of one layer step (TP = 1, gamma = 0.5) at c2 / c4 / c5, and of the
# Average / Same imputation kernels: time and DRAM / L2 bytes per launch (serialised, cold)
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum"
for c in c2 c4 c5; do
  CFG=$c timeout -s KILL 600 $NCU --metrics $M --clock-control none -k regex:'ztp_(select|gather|core|dw_reduce|splitk|expand|fill)' --csv python tools/one_step.py > gpurun_out/nongemm_$c.csv 2>&1
  CFG=$c timeout -s KILL 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv python tools/one_step.py > gpurun_out/launches_$c.csv 2>&1
done
for p in average same; do
  POLICY=$p timeout -s KILL 300 $NCU --metrics $M --clock-control none -k regex:'ztp_impute' --csv python tools/impute_one.py > gpurun_out/impute_$p.csv 2>&1
done
# full section set of the batched compaction kernel at c2 (3rd step)
CFG=c2 timeout -s KILL 600 $NCU --set full --import-source on --clock-control none -k regex:ztp_gather_multi -s 2 -c 1 -o gpurun_out/gather_multi_c2 -f python tools/one_step.py > gpurun_out/ncu_gather_full.log 2>&1
$NCU -i gpurun_out/gather_multi_c2.ncu-rep --page details > gpurun_out/gather_multi_c2_details.txt 2>&1
