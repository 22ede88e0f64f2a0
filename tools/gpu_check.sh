#!/bin/bash
# Full GPU check: all -m gpu tests, smoke(), default bench line (x2)
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3 | tee gpurun_out/gpu_tests.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke.txt
for i in 1 2; do timeout -s KILL 600 python bench.py 2>&1 | tail -1 > gpurun_out/bench_$i.txt
python -c "
import json;d=json.loads(open('gpurun_out/bench_$i.txt').read());print('run $i', 'ms/step %.4f'%d['ms_per_step'], 'TF %.1f'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'e2e %.1f'%d['e2e']['value'], d['clocks'])"; done
