"""Summarise an ncu launch list (--csv --log-file) of gpu__time_duration.sum and DRAM bytes:
per kernel, launches, mean per-launch time, share of kernel time, DRAM bytes per launch."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
ii = hdr.index("ID")
per = collections.defaultdict(dict)
names = {}
for r in rows[1:]:
    v = float(r[vi].replace(",", ""))
    unit = r[ui]
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3, "ms": 1e3,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
    per[r[ii]][r[mi]] = v * scale
    names[r[ii]] = r[ki]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for i, m in per.items():
    a = agg[names[i]]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values())
print(f"{len(per)} launches")
for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:56]:56s} n={n:3d} per-launch={t / n:9.1f} us  share={t / tot:.3f}  "
          f"dram/launch={b / n / 1e9:6.2f} GB ({b / t / 1e3:6.0f} GB/s)")
