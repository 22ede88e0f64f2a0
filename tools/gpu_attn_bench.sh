#!/bin/bash
# the layer step with the real attention core (NEXT-4) vs the stand-in, N = 1
mkdir -p gpurun_out
for c in c2 c4; do for a in standin real; do
timeout -s KILL 900 python bench.py --config $c --no-cpu --steps 100 --attention $a 2>&1 | tail -1 > gpurun_out/bench_attn_${c}_$a.txt
python -c "
import json;d=json.loads(open('gpurun_out/bench_attn_${c}_$a.txt').read());r=d['roofline'];print('$c $a', 'ms/step %.4f'%d['ms_per_step'], 'execTF %.1f'%d['value'], 'gemm_frac %.3f'%r['frac'], 'gemm_share %.3f'%r['gemm_share_of_step'], 'dense ms %.4f'%d['ms_dense_free'], 'speedup %.2f'%d['speedup_vs_dense'])" 2>&1 | tail -1
done; done | tee gpurun_out/attn_bench.txt
