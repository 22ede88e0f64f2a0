#!/bin/bash
# BWD order A/B: dX chain first + dW GEMMs last (ZTP_DW_LAST=1) vs per-linear concurrent dX/dW (default)
mkdir -p gpurun_out
ZTP_DW_LAST=1 timeout -s KILL 600 python -m pytest tests/test_gpu_layer.py -x -q -m gpu 2>&1 | tail -2 | tee gpurun_out/dwlast_tests.txt
ZTP_DW_LAST=1 timeout -s KILL 120 python tools/graph_timeline.py > gpurun_out/timeline_dwlast.txt 2>&1
tail -14 gpurun_out/timeline_dwlast.txt
for i in 1 2; do
ZTP_DW_LAST=1 timeout -s KILL 300 python bench.py --no-cpu 2>&1 | tail -1 > gpurun_out/bench_dwl1_$i.txt
ZTP_DW_LAST=0 timeout -s KILL 300 python bench.py --no-cpu 2>&1 | tail -1 > gpurun_out/bench_dwl0_$i.txt
done
python - <<'PY'
import json
for t in ("dwl1_1","dwl0_1","dwl1_2","dwl0_2"):
    try:
        d=json.loads(open(f"gpurun_out/bench_{t}.txt").read())
        print(t, "ms %.4f"%d["ms_per_step"], "TF %.1f"%d["value"], "gemm_frac %.3f"%d["roofline"]["frac"], "gemm_ms %.4f"%d["roofline"]["gemm_kernel_ms_per_step"], "launches", d["gpu_launches"], d.get("step_ms_dist"))
    except Exception as e:
        print(t, "ERR", e, open(f"gpurun_out/bench_{t}.txt").read()[:300])
PY
