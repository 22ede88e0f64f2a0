#!/bin/bash
# two-plane (GeLU / GeLU') epilogue with ping-pong staging: parity + FC1 FWD time in the step
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for i in 1 2; do timeout -s KILL 120 python tools/graph_timeline.py > gpurun_out/timeline_epi2_$i.txt 2>&1; sed -n '2,4p' gpurun_out/timeline_epi2_$i.txt; tail -1 gpurun_out/timeline_epi2_$i.txt; done
for i in 1 2; do timeout -s KILL 300 python bench.py --no-cpu 2>&1 | tail -1 > gpurun_out/bench_epi2.txt
python -c "
import json;d=json.loads(open('gpurun_out/bench_epi2.txt').read());print('run $i', 'ms/step %.4f'%d['ms_per_step'], 'gemm_frac %.3f'%d['roofline']['frac'], 'gemm_ms %.4f'%d['roofline']['gemm_kernel_ms_per_step'])"; done
