#!/bin/bash
# epilogue column spread (branch-free): parity, c4/c5 spread on/off, c4 CTA timeline
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests/test_gpu_layer.py -x -q -m gpu -k "c4 or schedule or c5 or c2_full_size_all" 2>&1 | tail -3 | tee gpurun_out/r2f_tests.txt
CONFIGS="c4 c5" bash tools/gpu_configs.sh; mv gpurun_out/configs.txt gpurun_out/configs_spread1.txt
ZTP_SPREAD_EPI=0 CONFIGS="c4 c5" bash tools/gpu_configs.sh; mv gpurun_out/configs.txt gpurun_out/configs_spread0.txt
CFG=c4 timeout -s KILL 300 python tools/cta_timeline.py > gpurun_out/c4_cta_spread.txt 2>&1
cat gpurun_out/configs_spread1.txt gpurun_out/configs_spread0.txt
