#!/bin/bash
# Round checkpoint 2: GPU tests, smoke, bench x3, ncu launch list + traffic + full capture, simulations
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
timeout -s KILL 120 python tools/graph_timeline.py > gpurun_out/timeline_final.txt 2>&1
bash tools/gpu_profiles.sh
timeout -s KILL 900 python tools/recovery_sim.py > gpurun_out/recovery_sim.log 2>&1
timeout -s KILL 900 python tools/adaptive_sim.py > gpurun_out/adaptive_sim.log 2>&1
timeout -s KILL 600 python tools/migration_table.py > gpurun_out/migration_table.log 2>&1
timeout -s KILL 600 python tools/lambda_sweep.py > gpurun_out/lambda_sweep.log 2>&1
tail -4 gpurun_out/adaptive_sim.log | cut -c1-200
