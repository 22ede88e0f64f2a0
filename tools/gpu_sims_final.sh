#!/bin/bash
# one-GPU recovery simulations with the final round-2 kernels: default cases, the c0 chi sweep, c5 adaptive
mkdir -p gpurun_out
OUT=gpurun_out/rs_final.json timeout -s KILL 1200 python tools/recovery_sim.py > gpurun_out/rs_final.log 2>&1
CASES=c0:8:1,c0:8:2,c0:8:3,c0:8:4,c0:8:6,c0:8:8,c0:8:4s,c0:8:8s OUT=gpurun_out/rs_c0_final.json timeout -s KILL 1500 python tools/recovery_sim.py > gpurun_out/rs_c0_final.log 2>&1
OUT=gpurun_out/as_c5_final.json timeout -s KILL 1500 python tools/adaptive_sim.py > gpurun_out/as_c5_final.log 2>&1
python - <<'PY'
import json
for f in ("gpurun_out/rs_final.json", "gpurun_out/rs_c0_final.json"):
    for r in json.load(open(f))["cases"]:
        print(r["config"], r["tp"], r["chi"], r["mode"], "recovery %.3f" % r["recovery"], r["final_plan"]["roles"])
for p in json.load(open("gpurun_out/as_c5_final.json"))["phases"]:
    print("c5 phase", p["phase"], "planned %.3f all %.3f" % (p["recovery_planned_steps"], p["recovery_all_steps"]), p["last_plan"]["roles"])
PY
