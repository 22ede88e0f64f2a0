#!/bin/bash
# paper-literal T_avg criterion (Eq.1): one-GPU recovery simulation at c2 TP=2/4, chi = 2
mkdir -p gpurun_out
CRIT=avg CASES=c2:2:2,c2:4:2,c3:4:2,c4:8:2 OUT=gpurun_out/recovery_sim_avg.json timeout -s KILL 1200 python tools/recovery_sim.py > gpurun_out/recovery_sim_avg.log 2>&1
grep '"config"' gpurun_out/recovery_sim_avg.log | cut -c1-400
