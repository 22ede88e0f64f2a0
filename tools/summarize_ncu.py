"""Summarise ncu --csv metric dumps: per kernel launch (last step of the
run) time, DRAM read / write, L2 bytes and achieved GB/s; usage:
python tools/summarize_ncu.py FILE [--last N]."""
import csv
import sys
from collections import OrderedDict


def load(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    if not rows:
        return []
    hdr = rows[0]
    iN, iV, iK, iKN = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID"), hdr.index("Kernel Name")
    iU = hdr.index("Metric Unit")
    d = OrderedDict()
    for r in rows[1:]:
        e = d.setdefault(r[iK], {"name": r[iKN]})
        v = float(r[iV].replace(",", ""))
        u = r[iU]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "us": 1e-6,
                 "usecond": 1e-6, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9,
                 "msecond": 1e-3}.get(u, 1)
        e[r[iN]] = v * scale
    return list(d.values())


def main():
    path = sys.argv[1]
    last = int(sys.argv[sys.argv.index("--last") + 1]) if "--last" in sys.argv else 0
    ks = load(path)
    if last:
        ks = ks[-last:]
    for k in ks:
        t = k.get("gpu__time_duration.sum", 0)
        rd, wr = k.get("dram__bytes_read.sum", 0), k.get("dram__bytes_write.sum", 0)
        l2 = k.get("lts__t_bytes.sum", 0)
        nm = k["name"].split("(")[0].replace("void ", "").replace("ztp::", "")[:34]
        extra = f"  dram r {rd / 1e6:7.2f} MB w {wr / 1e6:7.2f} MB ({(rd + wr) / t / 1e9 if t else 0:6.0f} GB/s)" \
                f"  L2 {l2 / 1e6:7.2f} MB" if rd or wr or l2 else ""
        print(f"{t * 1e6:8.2f} us  {nm:34s}{extra}")


if __name__ == "__main__":
    main()
