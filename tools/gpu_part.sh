#!/bin/bash
# concurrent dX/dW SM split: modelled (ZTP_PART=1) vs proportional with dW weight 1.2 / 1.0
mkdir -p gpurun_out
for i in 1 2; do
for v in "ZTP_PART=1" "ZTP_DW_SHARE=1.2" "ZTP_DW_SHARE=1.0"; do
env $v timeout -s KILL 300 python bench.py --no-cpu 2>&1 | tail -1 > gpurun_out/bench_part.txt
python -c "
import json;d=json.loads(open('gpurun_out/bench_part.txt').read());print('$v run $i', 'ms/step %.4f'%d['ms_per_step'], 'gemm_frac %.3f'%d['roofline']['frac'], 'gemm_ms %.4f'%d['roofline']['gemm_kernel_ms_per_step'])"
done; done | tee gpurun_out/part_ab.txt
ZTP_PART=1 timeout -s KILL 120 python tools/graph_timeline.py > gpurun_out/timeline_part1.txt 2>&1
ZTP_DW_SHARE=1.2 timeout -s KILL 120 python tools/graph_timeline.py > gpurun_out/timeline_share12.txt 2>&1
tail -13 gpurun_out/timeline_part1.txt; tail -13 gpurun_out/timeline_share12.txt
