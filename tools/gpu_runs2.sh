#!/bin/bash
# contiguous-run fast path in the batched compaction's 2D gathers: parity, configs, gather_multi times
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -2 | tee gpurun_out/runs2_tests.txt
CONFIGS="c2 c4 c5" bash tools/gpu_configs.sh > /dev/null 2>&1; cut -c1-175 gpurun_out/configs.txt
NCU=/usr/local/cuda/bin/ncu
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum"
for c in c2 c4 c5; do
  CFG=$c timeout -s KILL 600 $NCU --metrics $M --clock-control none -k regex:'ztp_(gather|expand)' --csv python tools/one_step.py > gpurun_out/runs2_$c.csv 2>&1
  echo "== $c"; python tools/summarize_ncu.py gpurun_out/runs2_$c.csv 2>&1 | tail -3
done
