#!/bin/bash
# cluster split-K check: GPU tests, bench, in-graph GEMM timeline, A/B vs ZTP_CSPLIT=0
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/gpu_tests.txt
cat gpurun_out/gpu_tests.txt
timeout -s KILL 120 python tools/graph_timeline.py > gpurun_out/timeline_cs1.txt 2>&1
ZTP_CSPLIT=0 timeout -s KILL 120 python tools/graph_timeline.py > gpurun_out/timeline_cs0.txt 2>&1
tail -14 gpurun_out/timeline_cs1.txt; tail -3 gpurun_out/timeline_cs0.txt
for i in 1 2; do
timeout -s KILL 300 python bench.py --no-cpu 2>&1 | tail -1 > gpurun_out/bench_cs1_$i.txt
ZTP_CSPLIT=0 timeout -s KILL 300 python bench.py --no-cpu 2>&1 | tail -1 > gpurun_out/bench_cs0_$i.txt
done
python - <<'PY'
import json
for t in ("cs1_1","cs0_1","cs1_2","cs0_2"):
    try:
        d=json.loads(open(f"gpurun_out/bench_{t}.txt").read())
        print(t, "ms %.4f"%d["ms_per_step"], "TF %.1f"%d["value"], "gemm_frac %.3f"%d["roofline"]["frac"], "gemm_ms %.4f"%d["roofline"]["gemm_kernel_ms_per_step"])
    except Exception as e:
        print(t, "ERR", e, open(f"gpurun_out/bench_{t}.txt").read()[:300])
PY
