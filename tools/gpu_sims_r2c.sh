#!/bin/bash
# one-GPU recovery simulations with the final round-2 kernels (library controller, modelled all-reduces)
mkdir -p gpurun_out
OUT=gpurun_out/recovery_sim_r2c.json timeout -s KILL 1500 python tools/recovery_sim.py > gpurun_out/recovery_sim_r2c.log 2>&1
OUT=gpurun_out/adaptive_sim_r2c.json timeout -s KILL 1500 python tools/adaptive_sim.py > gpurun_out/adaptive_sim_r2c.log 2>&1
tail -15 gpurun_out/recovery_sim_r2c.log; tail -12 gpurun_out/adaptive_sim_r2c.log
