"""Per-barrier-interval instruction / stall-sample split and top opcodes of one kernel of an ncu
report (--page source, SASS): where a phase-structured kernel (K5, K13) spends its issue slots.
usage: ncu_phases.py report.ncu-rep [kernel-index]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
which = int(sys.argv[2]) if len(sys.argv) > 2 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
secs = []
for line in out.splitlines():
    if line.startswith('"Kernel Name"'):
        secs.append([line])
    elif secs:
        secs[-1].append(line)
if not secs:
    sys.exit("no source page")
if which >= len(secs):
    sys.exit(1)            # no such kernel in the report (the caller's loop stops here)
sec = secs[which]
rows = list(csv.reader(sec[1:]))
hdr, data = rows[0], rows[1:]
ie = hdr.index("Instructions Executed")
ss = hdr.index("Warp Stall Sampling (All Samples)")
print(sec[0][:160])
tot_i = sum(int(r[ie] or 0) for r in data)
tot_s = sum(int(r[ss] or 0) for r in data)
print(f"warp-instructions {tot_i}, stall samples {tot_s}")
bars = [k for k, r in enumerate(data) if "BAR.SYNC" in r[1]]
edges = [0] + bars + [len(data)]
for a, b in zip(edges[:-1], edges[1:]):
    i = sum(int(data[k][ie] or 0) for k in range(a, b))
    s = sum(int(data[k][ss] or 0) for k in range(a, b))
    print(f"  SASS {a:5d}-{b:5d}: instructions {100 * i / tot_i:5.1f} %  stall samples {100 * s / tot_s:5.1f} %")
h = collections.Counter()
for r in data:
    op = [o for o in r[1].split() if not o.startswith("@")]
    if op:
        h[op[0].split(".")[0]] += int(r[ie] or 0)
print("top opcodes:", ", ".join(f"{k} {100 * v / tot_i:.1f}%" for k, v in h.most_common(12)))
