#!/bin/bash
# Zero tiles at a lineage row map: generic 16-byte stores (ZTP_ZERO_GENERIC=1) vs TMA scatter4 (=0)
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_kernels.py tests/test_gpu_runtime.py -x -q -m gpu 2>&1 | tail -2 | tee gpurun_out/zgen_tests.txt
NCU=/usr/local/cuda/bin/ncu
for zg in 1 0; do
  ZTP_ZERO_GENERIC=$zg CFG=c0 TP=8 GAMMAS=0.9 timeout -s KILL 600 $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:ztp --csv \
    --log-file gpurun_out/gov_c0_zg$zg.csv python tools/gamma_overhead.py > /dev/null 2>&1
  CFG=c0 TP=8 GAMMAS=0.9 python tools/gamma_overhead.py --parse gpurun_out/gov_c0_zg$zg.csv gpurun_out/gov_c0_zg$zg.json > gpurun_out/gov_c0_zg$zg.txt 2>&1
done
for rep in 1 2; do for zg in 1 0; do
  ZTP_ZERO_GENERIC=$zg CONFIGS="c2 c4" bash tools/gpu_configs.sh > /dev/null 2>&1
  sed "s/^/zg$zg rep$rep /" gpurun_out/configs.txt >> gpurun_out/zgen_ab.txt
done; done
paste gpurun_out/gov_c0_zg1.txt gpurun_out/gov_c0_zg0.txt | head -30; cat gpurun_out/zgen_ab.txt | cut -c1-200
