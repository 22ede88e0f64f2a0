#!/bin/bash
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
# sustained: a ~1.5 s timed region (power-capped clocks)
timeout -s KILL 600 python bench.py --steps 5000 --warmup 10 --no-cpu 2>&1 | tail -1 > gpurun_out/bench_sustained.txt
python -c "
import json;d=json.loads(open('gpurun_out/bench_sustained.txt').read());print('sustained', 'ms/step %.4f'%d['ms_per_step'], 'TF %.1f'%d['value'], 'frac %.3f'%d['roofline']['frac'], d['roofline']['peak'], d['roofline']['peak_source'], d['clocks'])"
# ncu full of the FC1 dW GEMM (8th GEMM launch of the profiled step: serial order dX, dW per linear)
timeout -s KILL 600 $NCU --set full --import-source on --clock-control none -k regex:ztp_gemm_kernel -s 31 -c 1 \
  -o gpurun_out/gemm_fc1_dw -f python tools/one_step.py > gpurun_out/ncu_fc1dw.log 2>&1
tail -1 gpurun_out/ncu_fc1dw.log
