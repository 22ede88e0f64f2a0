#!/bin/bash
# Interleaved A/B: for round in 1..R, each variant once; prints the headline
# ms_per_step followed by the repeat timings of phase C (BENCH_REPEAT).
mkdir -p gpurun_out
R=${R:-3}
: > gpurun_out/ab2.txt
for r in $(seq $R); do
  for v in "$@"; do
    out=$(env $v BENCH_REPEAT=3 timeout -s KILL 300 python bench.py --no-cpu --steps 300 2>&1)
    head=$(echo "$out" | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4f' % d['ms_per_step'])" 2>/dev/null)
    t=$(echo "$out" | grep repeat | awk '{print $4}' | tr '\n' ' ')
    echo "$v | head $head | $t" >> gpurun_out/ab2.txt
  done
done
