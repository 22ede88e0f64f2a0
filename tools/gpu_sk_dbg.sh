#!/bin/bash
mkdir -p gpurun_out
for sk in 0 1; do
ZTP_STREAMK=$sk timeout -s KILL 200 python tools/gemm_bench.py --shapes "2048,1024,8192;1024,2560,8192;1024,1024,8192" --gammas 0,0.5 > gpurun_out/gemm_bench_sk$sk.txt 2>&1
echo "== sk=$sk"; cat gpurun_out/gemm_bench_sk$sk.txt
done
ZTP_STREAMK=1 timeout -s KILL 300 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:ztp_gemm_kernel -s 3 -c 1 -o gpurun_out/sk_fwd -f python tools/gemm_bench.py --shapes "2048,1024,8192" --gammas 0 > gpurun_out/ncu_sk.log 2>&1
tail -3 gpurun_out/ncu_sk.log
