import csv, sys
rows = list(csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/launches.csv')))
hdr = None; data = []
for r in rows:
    if r and r[0] == 'ID': hdr = r; continue
    if hdr and len(r) == len(hdr): data.append(dict(zip(hdr, r)))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 22
tot = 0
for d in data[-n:]:
    v = float(d['Metric Value']) / 1000; tot += v
    print(f"{v:8.1f} us  {d['Kernel Name'][:70]}")
print('sum (serialized, cold)', round(tot, 1))
