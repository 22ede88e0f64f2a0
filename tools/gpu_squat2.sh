#!/bin/bash
# core BWD in stream order while a dW is pending (ZTP_SQUAT_GUARD=1, default) vs under PDL (=0), alternating, c2
mkdir -p gpurun_out
for rep in 1 2 3; do for v in 1 0; do
  ZTP_SQUAT_GUARD=$v CONFIGS="c2" bash tools/gpu_configs.sh > /dev/null 2>&1
  sed "s/^/guard$v rep$rep /" gpurun_out/configs.txt >> gpurun_out/squat2_ab.txt
done; done
ZTP_SQUAT_GUARD=0 CFG=c2 python tools/cta_timeline.py > gpurun_out/cta_c2_guard0.txt 2>&1
cut -c1-175 gpurun_out/squat2_ab.txt; tail -4 gpurun_out/cta_c2_guard0.txt
