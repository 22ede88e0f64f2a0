"""Summaries committed under profiles/: per-GEMM DRAM traffic of one step
(gemm_step.csv -> profiles/gemm_traffic.json + a table) and the key metrics of
the ncu --set full capture (gemm_fc2_fwd.ncu-rep)."""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"

rows = list(csv.reader(open(os.path.join(OUT, "gemm_step.csv"))))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6,
         "%": 1, "": 1}
per = {}
for d in data:
    v = float(d["Metric Value"].replace(",", "")) * SCALE.get(d.get("Metric Unit", ""), 1)
    per.setdefault(d["ID"], {"kernel": d["Kernel Name"][:40]})[d["Metric Name"]] = v   # bytes, ns, %
names = ["QKV fwd", "O fwd", "FC1 fwd (GeLU)", "FC2 fwd", "FC2 dX (GeLU')", "FC2 dW", "FC1 dX", "FC1 dW", "O dX", "O dW",
         "QKV dX", "QKV dW"]
lines = ["| # | GEMM | time us (cold) | DRAM read MB | DRAM write MB | tensor pipe % |", "|---|---|---|---|---|---|"]
tot = []
for i, (k, v) in enumerate(sorted(per.items(), key=lambda kv: int(kv[0]))):
    rd, wr = v.get("dram__bytes_read.sum", 0), v.get("dram__bytes_write.sum", 0)
    t = v.get("gpu__time_duration.sum", 0) / 1e3
    tp = v.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0)
    tot.append(rd + wr)
    lines.append(f"| {i} | {names[i] if i < len(names) else v['kernel']} | {t:.1f} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | {tp:.1f} |")
avg = sum(tot) / max(1, len(tot))
json.dump({"bytes_per_launch": avg, "per_launch_bytes": tot,
           "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over the 12 GEMM launches of one "
                     "c2 TP=1 gamma=0.5 step (tools/gpu_profiles.sh); bytes_per_launch = their mean"},
          open(os.path.join(ROOT, "profiles", "gemm_traffic.json"), "w"), indent=1)
open(os.path.join(ROOT, "profiles", f"{tag}_gemm_step_traffic.md"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines))

rep = os.path.join(OUT, "gemm_fc2_fwd.ncu-rep")
if os.path.exists(rep):
    raw = subprocess.run(["/usr/local/cuda/bin/ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    d = dict(zip(rr[0], rr[2] if len(rr) > 2 else rr[1]))
    units = dict(zip(rr[0], rr[1])) if len(rr) > 2 else {}
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
            "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__inst_executed.sum", "launch__grid_size", "launch__cluster_dim_x", "launch__registers_per_thread",
            "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second"]
    out = [f"# ncu --set full: FC2 FWD GEMM of one c2 TP=1 gamma=0.5 step ({tag})", ""]
    for k in keys:
        if k in d:
            out.append(f"{k}: {d[k]} {units.get(k, '')}")
    open(os.path.join(ROOT, "profiles", f"{tag}_ncu_full_fc2_fwd.txt"), "w").write("\n".join(out) + "\n")
    print("\n".join(out))
