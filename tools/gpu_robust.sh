#!/bin/bash
# robustness sweep: every config x odd prune ratios (short runs; failures only)
mkdir -p gpurun_out
for c in c1 c2 c3 c4 c5; do for g in 0.1 0.33 0.75 0.9; do
timeout -s KILL 300 python bench.py --config $c --gamma $g --steps 20 --warmup 3 --no-cpu > gpurun_out/rob_${c}_$g.log 2>&1
python -c "
import json
l=open('gpurun_out/rob_${c}_$g.log').read().strip().splitlines()[-1]
try:
    d=json.loads(l); print('$c $g OK ms %.4f TF %.1f'%(d['ms_per_step'], d['value']))
except Exception: print('$c $g FAIL', l[:300])"
done; done | tee gpurun_out/robust.txt
