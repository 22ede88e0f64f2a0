#!/bin/bash
# c0 round-robin straggler schedule (chi 2, 4, 8 on rotating ranks, then homogeneous) under the adaptive controller
mkdir -p gpurun_out
CFG=c0 SCHED=roundrobin OUT=gpurun_out/adaptive_sim_c0_rr.json timeout -s KILL 1500 python tools/adaptive_sim.py > gpurun_out/adaptive_sim_c0_rr.log 2>&1
tail -5 gpurun_out/adaptive_sim_c0_rr.log | cut -c1-400
