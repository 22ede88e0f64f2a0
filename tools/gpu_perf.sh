#!/bin/bash
# perf check: in-graph GEMM timeline + N=1 bench line (x2)
mkdir -p gpurun_out
timeout -s KILL 300 python tools/graph_timeline.py > gpurun_out/timeline.txt 2>&1
for i in 1 2; do timeout -s KILL 600 python bench.py --no-cpu 2>&1 | tail -1 > gpurun_out/bench_$i.txt
python -c "
import json;d=json.loads(open('gpurun_out/bench_$i.txt').read());r=d['roofline'];print('run $i', 'ms/step %.4f'%d['ms_per_step'], 'exec TF %.1f'%d['value'], 'method TF %.1f'%d['method_tflops'], 'gemm frac %.3f'%r['frac'], 'gemm ms %.4f'%r['gemm_kernel_ms_per_step'], 'share %.3f'%r['gemm_share_of_step'], d['clocks']['sm_mhz'])"; done | tee gpurun_out/perf.txt
