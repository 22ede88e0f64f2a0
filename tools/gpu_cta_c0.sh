#!/bin/bash
# per-CTA GEMM phases of a heavily resized straggler's step: c0 TP=8 rank at gamma 0 / 0.5 / 0.9
mkdir -p gpurun_out
for g in 0.0 0.5 0.9; do
  echo "== c0 TP=8 rank 0, gamma $g"; CFG=c0 TP=8 GAMMA=$g timeout -s KILL 300 python tools/cta_timeline.py 2>&1 | tail -13
done | tee gpurun_out/cta_c0_tp8.txt
