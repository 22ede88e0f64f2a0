#!/bin/bash
# stream-K hybrid GEMM schedule (ZTP_STREAMK=1, default) vs split-K + static (ZTP_STREAMK=0)
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/gpu_tests_sk.txt
cat gpurun_out/gpu_tests_sk.txt
ZTP_STREAMK=1 timeout -s KILL 120 python tools/graph_timeline.py > gpurun_out/timeline_sk1.txt 2>&1
tail -14 gpurun_out/timeline_sk1.txt
for i in 1 2; do
ZTP_STREAMK=1 timeout -s KILL 300 python bench.py --no-cpu 2>&1 | tail -1 > gpurun_out/bench_sk1_$i.txt
ZTP_STREAMK=0 timeout -s KILL 300 python bench.py --no-cpu 2>&1 | tail -1 > gpurun_out/bench_sk0_$i.txt
done
python - <<'PY'
import json
for t in ("sk1_1","sk0_1","sk1_2","sk0_2"):
    try:
        d=json.loads(open(f"gpurun_out/bench_{t}.txt").read())
        print(t, "ms %.4f"%d["ms_per_step"], "TF %.1f"%d["value"], "gemm_frac %.3f"%d["roofline"]["frac"], "gemm_ms %.4f"%d["roofline"]["gemm_kernel_ms_per_step"], "launches", d["gpu_launches"])
    except Exception as e:
        print(t, "ERR", e, open(f"gpurun_out/bench_{t}.txt").read()[:300])
PY
timeout -s KILL 900 python tools/adaptive_sim.py > gpurun_out/adaptive_sim.log 2>&1; echo rc=$? >> gpurun_out/adaptive_sim.log; tail -5 gpurun_out/adaptive_sim.log
