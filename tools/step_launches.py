"""One step of an ncu launch list (gpu__time_duration per kernel), the step
delimited by consecutive ztp_select launches."""
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
idx = [i for i, d in enumerate(data) if "select" in d["Kernel Name"]]
step = data[idx[-2]:idx[-1]]
tot = 0.0
for d in step:
    v = float(d["Metric Value"]) / 1000
    tot += v
    print(f"{v:7.1f} us  {d['Kernel Name'][:64]}")
print(f"step sum {tot:.1f} us over {len(step)} launches (serialized, cold)")
