#!/bin/bash
# pretest GPU test, one-GPU straggler simulations (recovery, lambda sweep, c5 adaptive), default bench line
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_pretest.py -x -q -m gpu 2>&1 | tail -3 | tee gpurun_out/pretest_test.txt
timeout -s KILL 900 python tools/recovery_sim.py > gpurun_out/recovery_sim.log 2>&1; echo rc=$? >> gpurun_out/recovery_sim.log
timeout -s KILL 600 python tools/lambda_sweep.py > gpurun_out/lambda_sweep.log 2>&1; echo rc=$? >> gpurun_out/lambda_sweep.log
timeout -s KILL 900 python tools/adaptive_sim.py > gpurun_out/adaptive_sim.log 2>&1; echo rc=$? >> gpurun_out/adaptive_sim.log
tail -5 gpurun_out/adaptive_sim.log
timeout -s KILL 300 python bench.py --no-cpu 2>&1 | tail -1 > gpurun_out/bench_base.txt
