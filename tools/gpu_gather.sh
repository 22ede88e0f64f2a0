#!/bin/bash
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -x -q -m gpu 2>&1 | tail -1
timeout -s KILL 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gather_multi --csv \
  --log-file gpurun_out/gather.csv python bench.py --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/gather.csv')) if len(r)>10]
h=rows[0]; d=rows[1:]
im=h.index('Metric Name'); iv=h.index('Metric Value'); iu=h.index('Metric Unit')
vals={}
for r in d: vals.setdefault(r[im],[]).append((float(r[iv].replace(',','')), r[iu]))
for k,v in vals.items(): print(k, v[-3:])
PY
for i in 1 2; do timeout -s KILL 300 python bench.py --no-cpu 2>&1 | tail -1 > gpurun_out/bench_g.txt; python -c "
import json;d=json.loads(open('gpurun_out/bench_g.txt').read());print('run $i', 'ms/step %.4f'%d['ms_per_step'], 'gemm_frac %.3f'%d['roofline']['frac'])"; done
