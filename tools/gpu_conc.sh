#!/bin/bash
# concurrent dX / dW with the SMs partitioned by work (ZTP_CONC=1) vs serial
mkdir -p gpurun_out
ZTP_CONC=1 timeout -s KILL 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/gpu_tests_conc.txt
cat gpurun_out/gpu_tests_conc.txt
ZTP_CONC=1 timeout -s KILL 120 python tools/graph_timeline.py > gpurun_out/timeline_conc1.txt 2>&1
tail -14 gpurun_out/timeline_conc1.txt
for i in 1 2; do
ZTP_CONC=1 timeout -s KILL 300 python bench.py --no-cpu 2>&1 | tail -1 > gpurun_out/bench_conc1_$i.txt
ZTP_CONC=0 timeout -s KILL 300 python bench.py --no-cpu 2>&1 | tail -1 > gpurun_out/bench_conc0_$i.txt
done
python - <<'PY'
import json
for t in ("conc1_1","conc0_1","conc1_2","conc0_2"):
    try:
        d=json.loads(open(f"gpurun_out/bench_{t}.txt").read())
        print(t, "ms %.4f"%d["ms_per_step"], "TF %.1f"%d["value"], "gemm_frac %.3f"%d["roofline"]["frac"], "gemm_ms %.4f"%d["roofline"]["gemm_kernel_ms_per_step"], "launches", d["gpu_launches"])
    except Exception as e:
        print(t, "ERR", e, open(f"gpurun_out/bench_{t}.txt").read()[:300])
PY
