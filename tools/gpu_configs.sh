#!/bin/bash
# bench line of every BASELINE config at N=1 (TP=1, homogeneous gamma=0.5)
mkdir -p gpurun_out
for c in ${CONFIGS:-c1 c2 c3 c4 c5}; do
timeout -s KILL 900 python bench.py --config $c --no-cpu --steps ${STEPS:-100} 2>&1 | tail -1 > gpurun_out/bench_cfg_$c.txt
python -c "
import json;d=json.loads(open('gpurun_out/bench_cfg_$c.txt').read());r=d['roofline'];print('$c', d['config']['workload'][:50], 'ms/step %.4f'%d['ms_per_step'], 'execTF %.1f'%d['value'], 'methodTF %.1f'%d['method_tflops'], 'gemm_frac %.3f'%r['frac'], 'gemm_share %.3f'%r['gemm_share_of_step'], 'dense ms %.4f'%d['ms_dense_free'], 'speedup %.2f'%d.get('speedup_vs_dense',0), 'clk', d['clocks']['sm_mhz'])" 2>&1 | tail -1
done | tee gpurun_out/configs.txt
