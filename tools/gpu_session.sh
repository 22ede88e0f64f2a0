#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -x -q -m gpu 2>&1 | tail -15 | tee gpurun_out/gpu_tests.txt
timeout -s KILL 200 python tools/gemm_bench.py --shapes "1024,4096,8192;4096,1024,8192;1024,1024,8192" --gammas 0,0.5 2>&1 | tee gpurun_out/gemm_bench.txt
timeout -s KILL 300 python bench.py --no-cpu 2>&1 | tail -1 | tee gpurun_out/bench.txt
