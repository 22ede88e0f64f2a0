#!/bin/bash
# layer parity (migration paths), one-GPU straggler simulations, Table I analog, default bench line
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_layer.py tests/test_pretest.py -x -q -m gpu 2>&1 | tail -3 | tee gpurun_out/layer_tests.txt
timeout -s KILL 900 python tools/recovery_sim.py > gpurun_out/recovery_sim.log 2>&1; echo rc=$? >> gpurun_out/recovery_sim.log
timeout -s KILL 600 python tools/migration_table.py > gpurun_out/migration_table.log 2>&1; echo rc=$? >> gpurun_out/migration_table.log
tail -12 gpurun_out/migration_table.log
timeout -s KILL 900 python tools/adaptive_sim.py > gpurun_out/adaptive_sim.log 2>&1; echo rc=$? >> gpurun_out/adaptive_sim.log
tail -5 gpurun_out/adaptive_sim.log | cut -c1-300
timeout -s KILL 600 python tools/lambda_sweep.py > gpurun_out/lambda_sweep.log 2>&1; echo rc=$? >> gpurun_out/lambda_sweep.log
timeout -s KILL 300 python bench.py --no-cpu 2>&1 | tail -1 > gpurun_out/bench_base.txt
