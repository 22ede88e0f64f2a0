#!/bin/bash
# one change, checked: parity (kernels + layer), per-CTA and in-graph GEMM timelines, 3 bench runs
mkdir -p gpurun_out
T=${TAG:-chk}
timeout -s KILL 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -x -q -m gpu 2>&1 | tail -3 > gpurun_out/${T}_tests.txt
timeout -s KILL 300 python tools/cta_timeline.py > gpurun_out/${T}_cta.txt 2>&1
timeout -s KILL 300 python tools/graph_timeline.py > gpurun_out/${T}_graph.txt 2>&1
for i in 1 2 3; do timeout -s KILL 300 python bench.py --no-cpu --steps 300 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4f' % d['ms_per_step'], d['clocks']['sm_mhz'])"; done > gpurun_out/${T}_bench.txt 2>&1
cat gpurun_out/${T}_tests.txt gpurun_out/${T}_bench.txt; tail -1 gpurun_out/${T}_graph.txt
