#!/bin/bash
# bench line of every BASELINE config at N=1 (TP=1, homogeneous gamma=0.5)
mkdir -p gpurun_out
for c in c1 c2 c3 c4 c5; do
timeout -s KILL 600 python bench.py --config $c --no-cpu 2>&1 | tail -1 > gpurun_out/bench_cfg_$c.txt
python -c "
import json;d=json.loads(open('gpurun_out/bench_cfg_$c.txt').read());print('$c', d['config']['workload'][:60], 'ms/step %.4f'%d['ms_per_step'], 'TF %.1f'%d['value'], 'gemm_frac %.3f'%d['roofline']['frac'], 'dense ms %.4f'%d['ms_dense_free'], 'speedup %.2f'%d.get('speedup_vs_dense',0))" 2>&1 | tail -1
done | tee gpurun_out/configs.txt
