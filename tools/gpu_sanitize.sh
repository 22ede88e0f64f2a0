#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over the c1 layer step (TP = 1, gamma = 0.5, 3 steps)
# and over a c2-shaped GEMM of each kind; summaries into gpurun_out/sanitize_*.txt
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  CFG=c1 STEPS=1 timeout -s KILL 900 $CS --tool $tool --print-limit 20 python tools/one_step.py > gpurun_out/sanitize_c1_$tool.txt 2>&1
  tail -3 gpurun_out/sanitize_c1_$tool.txt
done
K=512 NN=1024 TOK=1024 timeout -s KILL 900 $CS --tool memcheck --print-limit 20 python tools/ncu_gemm.py > gpurun_out/sanitize_gemm_memcheck.txt 2>&1
tail -3 gpurun_out/sanitize_gemm_memcheck.txt
ACT=gelu K=512 NN=1024 TOK=1024 timeout -s KILL 900 $CS --tool racecheck --print-limit 20 python tools/ncu_gemm.py > gpurun_out/sanitize_gemm_racecheck.txt 2>&1
tail -3 gpurun_out/sanitize_gemm_racecheck.txt
