#!/bin/bash
# Round checkpoint: all GPU tests, smoke, bench (3 runs), ncu launch list + per-GEMM traffic + one full capture,
# the one-GPU simulations.
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3 | tee gpurun_out/gpu_tests.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke.txt
for i in 1 2 3; do timeout -s KILL 600 python bench.py 2>&1 | tail -1 > gpurun_out/bench_final_$i.txt; done
python - <<'PY'
import json
for i in (1,2,3):
    d=json.loads(open(f"gpurun_out/bench_final_{i}.txt").read())
    print(i, "ms %.4f"%d["ms_per_step"], "TF %.1f"%d["value"], "frac %.3f"%d["roofline"]["frac"], "e2e %.1f"%d["e2e"]["value"], d["clocks"])
PY
bash tools/gpu_profiles.sh
timeout -s KILL 900 python tools/recovery_sim.py > gpurun_out/recovery_sim.log 2>&1
timeout -s KILL 900 python tools/adaptive_sim.py > gpurun_out/adaptive_sim.log 2>&1
tail -4 gpurun_out/adaptive_sim.log | cut -c1-200
