#!/bin/bash
# end-of-round evidence: homogeneous gamma sweep at TP=1 (E2 analog) and a sustained bench (5000 steps, power-capped)
mkdir -p gpurun_out
bash tools/gpu_gamma.sh
timeout -s KILL 900 python bench.py --steps 5000 --warmup 50 --no-cpu 2>&1 | tail -1 > gpurun_out/bench_sustained.txt
python -c "
import json;d=json.loads(open('gpurun_out/bench_sustained.txt').read());r=d['roofline'];print('sustained', 'ms/step %.4f'%d['ms_per_step'], 'TF %.1f'%d['value'], 'frac %.3f'%r['frac'], 'peak', r['peak'], r['peak_source'], d['clocks'])"
