#!/bin/bash
# c0 (ViT-1B, the paper's shape): parity at TP=8, bench line at TP=1, and the E4-analog chi sweep (one-GPU simulation)
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_layer.py -q -m gpu -k c0 2>&1 | tail -2 | tee gpurun_out/c0_tests.txt
CONFIGS="c0" bash tools/gpu_configs.sh
CASES=c0:8:1,c0:8:2,c0:8:3,c0:8:4,c0:8:6,c0:8:8,c0:8:4s,c0:8:8s OUT=gpurun_out/recovery_sim_c0_chi.json timeout -s KILL 2400 python tools/recovery_sim.py > gpurun_out/recovery_sim_c0_chi.log 2>&1
grep '"config"' gpurun_out/recovery_sim_c0_chi.log | cut -c1-330
