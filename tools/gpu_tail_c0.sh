#!/bin/bash
# FWD tail halves at a TP = 8 rank (c0): few-tile FWD GEMMs run on twice the pairs; per-CTA phases and recovery
mkdir -p gpurun_out
for v in 1 0; do
  echo "== TAIL_HALVES=$v c0 TP=8 gamma 0.5"; ZTP_TAIL_HALVES=$v CFG=c0 TP=8 GAMMA=0.5 timeout -s KILL 300 python tools/cta_timeline.py 2>&1 | head -6
  ZTP_TAIL_HALVES=$v CASES=c0:8:2,c0:8:3,c2:4:2 OUT=gpurun_out/rs_tail$v.json timeout -s KILL 900 python tools/recovery_sim.py 2>&1 | grep '"config"' | cut -c1-230 | sed "s/^/tail$v /"
done
