#!/bin/bash
# SURVEY §8(d) c2 TP=1 homogeneous gamma sweep {0, 1/4, 1/2, 9/10} (E2 analog), and c4
mkdir -p gpurun_out
for c in c2 c4; do for g in 0 0.25 0.5 0.9; do
timeout -s KILL 600 python bench.py --config $c --gamma $g --no-cpu 2>&1 | tail -1 > gpurun_out/bench_g_${c}_$g.txt
python -c "
import json;d=json.loads(open('gpurun_out/bench_g_${c}_$g.txt').read());print('$c gamma $g', 'ms/step %.4f'%d['ms_per_step'], 'TF %.1f'%d['value'], 'gemm_frac %.3f'%d['roofline']['frac'], 'dense ms %.4f'%d['ms_dense_free'], 'speedup %.2f'%d.get('speedup_vs_dense',0))" 2>&1 | tail -1
done; done | tee gpurun_out/gamma_sweep.txt
