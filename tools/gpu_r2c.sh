#!/bin/bash
# round 2: GPU tests, bench N=1, bench N=2/4 on one shared GPU (path validation)
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 > gpurun_out/gpu_tests.txt
timeout -s KILL 600 python bench.py 2>&1 | tail -3 > gpurun_out/bench_1.txt
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --share-gpu --config c1 > gpurun_out/bench_share2_c1.txt 2>&1
timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --steps 5 --warmup 3 --share-gpu --config c1 --ctl-steps 4 > gpurun_out/bench_share4_c1.txt 2>&1
