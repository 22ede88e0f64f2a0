#!/bin/bash
# One GPU session: build check, GPU parity tests, GEMM micro-bench.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > gpurun_out/smi.txt 2>&1
python -c "import paper_2401_11469_b200 as z; print(z.ztp_version())"
timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu 2>&1 | tail -40 | tee gpurun_out/gpu_tests.txt
timeout -s KILL 300 python tools/gemm_bench.py 2>&1 | tee gpurun_out/gemm_bench.txt
