#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3 | tee gpurun_out/smoke.txt
timeout -s KILL 600 python bench.py 2>&1 | tail -5 | tee gpurun_out/bench.txt
