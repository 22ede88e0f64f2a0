#!/bin/bash
# round 2 baseline: GPU tests, smoke, default bench line
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 > gpurun_out/gpu_tests.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 > gpurun_out/smoke.txt
timeout -s KILL 600 python bench.py 2>&1 | tail -1 > gpurun_out/bench_1.txt
