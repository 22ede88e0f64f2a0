#!/bin/bash
# O projection's dW after the core, beside the QKV backward (ZTP_LATE_O_DW=1) vs beside its own dX (=0)
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_layer.py -x -q -m gpu -k "schedule" 2>&1 | tail -2 | tee gpurun_out/lateo_tests.txt
for rep in 1 2 3; do for v in 1 0; do
  ZTP_LATE_O_DW=$v CONFIGS="c2 c4" bash tools/gpu_configs.sh > /dev/null 2>&1
  sed "s/^/late$v rep$rep /" gpurun_out/configs.txt >> gpurun_out/lateo_ab.txt
done; done
ZTP_LATE_O_DW=1 CFG=c2 python tools/cta_timeline.py > gpurun_out/cta_c2_late1.txt 2>&1
ZTP_LATE_O_DW=0 CFG=c2 python tools/cta_timeline.py > gpurun_out/cta_c2_late0.txt 2>&1
cut -c1-175 gpurun_out/lateo_ab.txt; tail -5 gpurun_out/cta_c2_late1.txt; tail -5 gpurun_out/cta_c2_late0.txt
