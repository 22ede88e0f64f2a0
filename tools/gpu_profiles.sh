#!/bin/bash
# Round profiles: launch list of the bench command, per-GEMM DRAM bytes of one
# step, and one ncu --set full capture of the largest GEMM (FC2 FWD).
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout -s KILL 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_bench.log 2>&1
# one step's 12 GEMM launches (after 2 warm-up steps = 24 launches)
timeout -s KILL 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
  --clock-control none -k regex:ztp_gemm_kernel -s 24 -c 12 --csv --log-file gpurun_out/gemm_step.csv \
  python tools/one_step.py > gpurun_out/ncu_step.log 2>&1
# full section set on the FC2 FWD GEMM of that step (4th GEMM launch)
timeout -s KILL 600 $NCU --set full --import-source on --clock-control none -k regex:ztp_gemm_kernel -s 27 -c 1 \
  -o gpurun_out/gemm_fc2_fwd -f python tools/one_step.py > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
