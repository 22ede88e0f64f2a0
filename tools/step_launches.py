"""One step of an ncu launch list (gpu__time_duration per kernel), the step
delimited by consecutive ztp_select launches (round 1), or by consecutive
batched compactions (ztp_gather_multi opens every step since the selection
runs once per plan, A-46)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv")))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
from collections import Counter
idx = [i for i, d in enumerate(data) if "gather_multi" in d["Kernel Name"]]
if len(idx) < 2:
    idx = [i for i, d in enumerate(data) if "select" in d["Kernel Name"]]
# the step = the most common distance between consecutive delimiters (>= 8
# launches), its last occurrence
segs = [(idx[i], idx[i + 1]) for i in range(len(idx) - 1) if idx[i + 1] - idx[i] >= 8]
n = Counter(b - a for a, b in segs).most_common(1)[0][0]
a, b = [sg for sg in segs if sg[1] - sg[0] == n][-1]
step = data[a:b]
tot = 0.0
for d in step:
    v = float(d["Metric Value"]) / 1000
    tot += v
    print(f"{v:7.1f} us  {d['Kernel Name'][:64]}")
print(f"step sum {tot:.1f} us over {len(step)} launches (serialized, cold)")
