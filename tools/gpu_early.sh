#!/bin/bash
# A-operand early prefetch: parity (layer / kernels / peer tests), the per-CTA
# timeline and the in-graph GEMM timeline with and without, interleaved bench A/B
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_kernels.py tests/test_gpu_peer.py -x -q -m gpu 2>&1 | tail -4 | tee gpurun_out/early_tests.txt
for v in 0 1; do
  ZTP_A_EARLY=$v timeout -s KILL 300 python tools/cta_timeline.py > gpurun_out/early_cta_$v.txt 2>&1
  ZTP_A_EARLY=$v timeout -s KILL 300 python tools/graph_timeline.py > gpurun_out/early_graph_$v.txt 2>&1
done
tail -3 gpurun_out/early_graph_*.txt
R=3 bash tools/gpu_ab2.sh ZTP_A_EARLY=0 ZTP_A_EARLY=1
cat gpurun_out/ab2.txt
