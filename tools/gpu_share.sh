#!/bin/bash
# concurrent dX/dW SM split: weight of dW's work (ZTP_DW_SHARE) sweep, alternating
mkdir -p gpurun_out
for i in 1 2; do
for sh in 1.0 1.2 1.4 1.1; do
ZTP_DW_SHARE=$sh timeout -s KILL 300 python bench.py --no-cpu 2>&1 | tail -1 > gpurun_out/bench_share_${sh}_$i.txt
python -c "
import json;d=json.loads(open('gpurun_out/bench_share_${sh}_$i.txt').read());print('share $sh run $i', 'ms/step %.4f'%d['ms_per_step'], 'gemm_frac %.3f'%d['roofline']['frac'], 'gemm_ms %.4f'%d['roofline']['gemm_kernel_ms_per_step'])"
done; done | tee gpurun_out/share_sweep.txt
