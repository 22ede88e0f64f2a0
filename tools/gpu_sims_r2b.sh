#!/bin/bash
mkdir -p gpurun_out
CASES=c4:8:3s OUT=gpurun_out/recovery_sim_r2b.json timeout -s KILL 1200 python tools/recovery_sim.py > gpurun_out/recovery_sim_r2b.log 2>&1
OUT=gpurun_out/adaptive_sim_r2b.json timeout -s KILL 1500 python tools/adaptive_sim.py > gpurun_out/adaptive_sim_r2b.log 2>&1
