#!/bin/bash
# ncu --set full of the FC1 dW and QKV dW GEMMs of the c2 TP=1 gamma=0.5 step
# (launch 31 and 35 of tools/one_step.py: 2 warm-up steps x 12 GEMMs first),
# plus tests of the new gather / expand kernels and the cluster split-K option
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout -s KILL 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/gpu_tests.txt
ZTP_CSPLIT=1 timeout -s KILL 600 python -m pytest tests/test_gpu_layer.py -m gpu -x -q 2>&1 | tail -3 > gpurun_out/gpu_tests_csplit.txt
cat gpurun_out/gpu_tests.txt gpurun_out/gpu_tests_csplit.txt
for k in 31 35; do
timeout -s KILL 600 $NCU --set full --import-source on --clock-control none -k regex:ztp_gemm_kernel -s $k -c 1 \
  -o gpurun_out/gemm_dw_$k -f python tools/one_step.py > gpurun_out/ncu_dw_$k.log 2>&1
tail -1 gpurun_out/ncu_dw_$k.log
done
for c in "c4 8"; do set -- $c
  CFG=$1 TP=$2 timeout -s KILL 400 $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:ztp --csv \
    --log-file gpurun_out/gov_$1_$2.csv python tools/gamma_overhead.py > gpurun_out/gov_$1_$2.log 2>&1
  CFG=$1 TP=$2 python tools/gamma_overhead.py --parse gpurun_out/gov_$1_$2.csv gpurun_out/gov_$1_$2.json > gpurun_out/gov_$1_$2.txt 2>&1
done
grep -v "gemm_kernel" gpurun_out/gov_c4_8.txt | head -40
