"""Cut an ncu launch list (gpu__time_duration.sum, dram__bytes_read/write.sum; one warm-up and
one measured call per record, tools/config_calls.py) into calls and write {key: {"bytes": DRAM
bytes of the measured call, "ms": its summed kernel time, "kernels": [...]}} (FGF_NCU_BYTES of
tests/test_report_gpu.py).  usage: ncu_bytes.py launches.csv calls.json out.json"""
import collections
import csv
import json
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ui, ii = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                      hdr.index("Metric Unit"), hdr.index("ID"))
per = collections.OrderedDict()
for r in rows[1:]:
    v = float(r[vi].replace(",", ""))
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r[ui], 1.0)
    d = per.setdefault(int(r[ii]), {"name": r[ki]})
    d[r[mi]] = v * scale
launches = [per[k] for k in sorted(per)]
calls = json.load(open(sys.argv[2]))
res, pos = {}, 0
for c in calls:
    n = c["launches"]
    meas = launches[pos + n: pos + 2 * n]
    pos += 2 * n
    res[c["key"]] = {
        "bytes": sum(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0) for m in meas),
        "ms": sum(m.get("gpu__time_duration.sum", 0) for m in meas),
        "kernels": [(m["name"][:60], round(m.get("gpu__time_duration.sum", 0), 5),
                     m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) for m in meas]}
assert pos == len(launches), (pos, len(launches))
json.dump(res, open(sys.argv[3], "w"), indent=1)
print(json.dumps({k: (v["bytes"], round(v["ms"], 4)) for k, v in res.items()}))
