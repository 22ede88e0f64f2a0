#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 900 python tools/adaptive_sim.py > gpurun_out/adaptive_sim.log 2>&1; echo rc=$? >> gpurun_out/adaptive_sim.log
tail -5 gpurun_out/adaptive_sim.log | cut -c1-250
timeout -s KILL 900 python tools/recovery_sim.py > gpurun_out/recovery_sim2.log 2>&1; cp gpurun_out/recovery_sim.json gpurun_out/recovery_sim_rep2.json
python - <<'PY'
import json
d=json.load(open('gpurun_out/recovery_sim_rep2.json'))
for c in d['cases']:
    print(c['config'], c['tp'], c['chi'], c['plan'], round(c['T_free_ms'],3), round(c['T_unbal_ms'],3), round(c['first_plan']['T_bal_ms'],3), round(c['T_bal_ms'],3), round(c['recovery_compute'],3), round(c['recovery_with_comm'],3))
PY
