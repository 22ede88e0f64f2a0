#!/bin/bash
# A/B bench runs: each variant (env assignments) twice, one JSON line each
mkdir -p gpurun_out
: > gpurun_out/ab.txt
for v in "$@"; do
  for i in 1 2; do
    echo -n "$v | " >> gpurun_out/ab.txt
    env $v timeout -s KILL 300 python bench.py --no-cpu 2>&1 | tail -1 >> gpurun_out/ab.txt
  done
done
