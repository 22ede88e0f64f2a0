#!/bin/bash
# A/B: 3 epilogue staging buffers + 4-stage ring (libztp.so) vs 2 + 5 (libztp_stg2.so), alternating
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_kernels.py -x -q -m gpu 2>&1 | tail -2 | tee gpurun_out/stg3_tests.txt
cp paper_2401_11469_b200/libztp.so /tmp/libztp_stg3.so
for rep in 1 2; do
  for v in stg3 stg2; do
    if [ $v = stg3 ]; then cp /tmp/libztp_stg3.so paper_2401_11469_b200/libztp.so; else cp paper_2401_11469_b200/libztp_stg2.so paper_2401_11469_b200/libztp.so; fi
    CONFIGS="c2 c4" bash tools/gpu_configs.sh > /dev/null 2>&1
    sed "s/^/$v rep$rep /" gpurun_out/configs.txt >> gpurun_out/stg3_ab.txt
    CFG=c2 timeout -s KILL 300 python tools/cta_timeline.py > gpurun_out/cta_c2_$v.txt 2>&1
  done
done
cat gpurun_out/stg3_ab.txt
