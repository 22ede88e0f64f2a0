#!/bin/bash
# column spread kernels (staged expand_cols, L1 gathers in dw_reduce): parity, ncu per kernel, step timeline, configs
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -x -q -m gpu 2>&1 | tail -3 | tee gpurun_out/spread_tests.txt
NCU=/usr/local/cuda/bin/ncu
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum"
for c in c2 c4 c5; do
  CFG=$c timeout -s KILL 600 $NCU --metrics $M --clock-control none -k regex:'ztp_(dw_reduce|splitk|expand|gather)' --csv python tools/one_step.py > gpurun_out/spread_$c.csv 2>&1
  python tools/summarize_ncu.py gpurun_out/spread_$c.csv --last 8 > gpurun_out/spread_$c.txt 2>&1
done
timeout -s KILL 300 python tools/graph_timeline.py > gpurun_out/spread_graph.txt 2>&1
CONFIGS="c2 c4 c5" bash tools/gpu_configs.sh
