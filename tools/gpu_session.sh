#!/bin/bash
# One GPU session: GPU parity tests + GEMM micro-bench.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > gpurun_out/smi.txt 2>&1
timeout -s KILL 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -40 | tee gpurun_out/gpu_tests.txt
timeout -s KILL 300 python tools/gemm_bench.py 2>&1 | tee gpurun_out/gemm_bench.txt
ZTP_GATHER4=1 timeout -s KILL 300 python tools/gemm_bench.py --shapes "1024,4096,8192" --gammas 0.5 2>&1 | tee gpurun_out/gemm_bench_g4.txt
