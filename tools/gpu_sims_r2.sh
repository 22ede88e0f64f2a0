#!/bin/bash
# round 2: GPU tests, then the one-GPU controller simulations with the current kernels
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -3 > gpurun_out/gpu_tests.txt
CASES=c2:2:2,c2:4:2,c3:4:2,c4:8:2,c4:8:3s OUT=gpurun_out/recovery_sim_r2.json timeout -s KILL 1500 python tools/recovery_sim.py > gpurun_out/recovery_sim_r2.log 2>&1
OUT=gpurun_out/adaptive_sim_r2.json timeout -s KILL 1200 python tools/adaptive_sim.py > gpurun_out/adaptive_sim_r2.log 2>&1
