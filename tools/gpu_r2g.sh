#!/bin/bash
# column spread over the lineage rows (Zero rows written, not read; no Zero units in the dW GEMM)
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests/test_gpu_layer.py tests/test_gpu_kernels.py -x -q -m gpu 2>&1 | tail -3 | tee gpurun_out/r2g_tests.txt
CONFIGS="c4 c5 c2" bash tools/gpu_configs.sh
