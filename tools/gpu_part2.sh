#!/bin/bash
# dX/dW partition with the epilogue / Zero-tile term (ZTP_PART=1) vs MMA-only (=2): c0 TP=8 rank timelines,
# bench configs (alternating), and the c0 chi sweep (one-GPU recovery simulation)
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_runtime.py -x -q -m gpu 2>&1 | tail -2 | tee gpurun_out/part2_tests.txt
for pm in 1 2; do for g in 0.5 0.9; do
  echo "== PART=$pm c0 TP=8 gamma $g"; ZTP_PART=$pm CFG=c0 TP=8 GAMMA=$g timeout -s KILL 300 python tools/cta_timeline.py 2>&1 | tail -13
done; done > gpurun_out/part2_cta.txt
for rep in 1 2; do for pm in 1 2; do
  ZTP_PART=$pm CONFIGS="c2 c4" bash tools/gpu_configs.sh > /dev/null 2>&1
  sed "s/^/part$pm rep$rep /" gpurun_out/configs.txt >> gpurun_out/part2_ab.txt
done; done
for pm in 1 2; do
  ZTP_PART=$pm CASES=c0:8:2,c0:8:3,c0:8:4,c2:4:2,c4:8:2 OUT=gpurun_out/rs_part$pm.json timeout -s KILL 1200 python tools/recovery_sim.py 2>&1 | grep '"config"' | cut -c1-260 | sed "s/^/part$pm /" >> gpurun_out/part2_rs.txt
done
cat gpurun_out/part2_ab.txt | cut -c1-170; cat gpurun_out/part2_rs.txt
