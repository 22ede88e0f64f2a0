mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_pretest.py -x -q -m gpu 2>&1 | tail -5 | tee gpurun_out/pretest_test.txt
timeout -s KILL 900 python tools/adaptive_sim.py > gpurun_out/adaptive_sim.log 2>&1; echo rc=$? >> gpurun_out/adaptive_sim.log
tail -8 gpurun_out/adaptive_sim.log
