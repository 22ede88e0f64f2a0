#!/bin/bash
# round 2: GPU tests, smoke, controller-driven recovery simulation
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 > gpurun_out/gpu_tests.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 > gpurun_out/smoke.txt
CASES=c2:2:2,c4:8:2,c4:8:3s timeout -s KILL 900 python tools/recovery_sim.py > gpurun_out/recovery_sim.log 2>&1
