#!/bin/bash
# core BWD launched in stream order while a concurrent dW is pending (ZTP_SQUAT_GUARD=1) vs under PDL
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for i in 1 2; do
for v in "ZTP_SQUAT_GUARD=3" "ZTP_SQUAT_GUARD=1" "ZTP_SQUAT_GUARD=0"; do
env $v timeout -s KILL 300 python bench.py --no-cpu 2>&1 | tail -1 > gpurun_out/bench_sq.txt
python -c "
import json;d=json.loads(open('gpurun_out/bench_sq.txt').read());print('$v run $i', 'ms/step %.4f'%d['ms_per_step'], 'gemm_frac %.3f'%d['roofline']['frac'], 'gemm_ms %.4f'%d['roofline']['gemm_kernel_ms_per_step'])"
done; done | tee gpurun_out/squat_ab.txt
ZTP_SQUAT_GUARD=1 timeout -s KILL 120 python tools/graph_timeline.py > gpurun_out/timeline_squat1.txt 2>&1
tail -13 gpurun_out/timeline_squat1.txt
