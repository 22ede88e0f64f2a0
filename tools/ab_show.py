import json, sys
for l in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ab.txt"):
    v, j = l.split(" | ", 1)
    try:
        d = json.loads(j)
        print(f"{v:28s} step {d['ms_per_step']*1e3:6.1f} us  dense {d['ms_dense_free']*1e3:6.1f} us  e2e {d['e2e']['ms_per_step']*1e3:6.1f} us  {d['value']:6.1f} TF/s")
    except Exception as e:
        print(v, "ERR", j[:200])
