#!/bin/bash
# FWD tail halves (ZTP_TAIL_HALVES=1) vs whole tiles (=0): parity, bench A/B alternating, c2 CTA timeline
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -2 | tee gpurun_out/tail_tests.txt
for rep in 1 2 3; do for v in 1 0; do
  ZTP_TAIL_HALVES=$v CONFIGS="c2 c4" bash tools/gpu_configs.sh > /dev/null 2>&1
  sed "s/^/tail$v rep$rep /" gpurun_out/configs.txt >> gpurun_out/tail_ab.txt
done; done
ZTP_TAIL_HALVES=1 CFG=c2 python tools/cta_timeline.py > gpurun_out/cta_c2_tail1.txt 2>&1
ZTP_TAIL_HALVES=0 CFG=c2 python tools/cta_timeline.py > gpurun_out/cta_c2_tail0.txt 2>&1
cut -c1-175 gpurun_out/tail_ab.txt; head -5 gpurun_out/cta_c2_tail1.txt; head -5 gpurun_out/cta_c2_tail0.txt
