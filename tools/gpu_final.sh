#!/bin/bash
# round-2 checkpoint: smoke, default bench (x2), reference arm, ncu launch list of the bench command
mkdir -p gpurun_out
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 > gpurun_out/smoke.txt
for i in 1 2; do timeout -s KILL 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench_$i.txt; done
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_ref.txt
NCU=/usr/local/cuda/bin/ncu
timeout -s KILL 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_bench.log 2>&1
tail -2 gpurun_out/ncu_bench.log
