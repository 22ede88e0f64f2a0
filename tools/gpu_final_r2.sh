#!/bin/bash
# Round-2 evidence: all GPU tests, smoke, default bench x2, every config's bench line, the ncu launch
# list of the bench command + per-GEMM step traffic + ncu full of FC2 FWD, non-GEMM kernels at c4/c5
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -q -m gpu 2>&1 | tail -3 | tee gpurun_out/gpu_tests.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | tee gpurun_out/smoke.txt
for i in 1 2; do timeout -s KILL 600 python bench.py 2>&1 | tail -1 > gpurun_out/bench_$i.txt; done
CONFIGS="c2 c3 c4 c5" bash tools/gpu_configs.sh
bash tools/gpu_profiles.sh
NCU=/usr/local/cuda/bin/ncu
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum"
for c in c4 c5; do
  CFG=$c timeout -s KILL 600 $NCU --metrics $M --clock-control none -k regex:'ztp_(gather|core|dw_reduce|splitk|expand)' --csv python tools/one_step.py > gpurun_out/nongemm_$c.csv 2>&1
done
