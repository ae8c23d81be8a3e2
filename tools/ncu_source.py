import csv, sys, subprocess
rep, which = sys.argv[1], int(sys.argv[2])
ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
lines = out.splitlines()
secs = []
for l in lines:
    if l.startswith('"Kernel Name"'):
        secs.append([l])
    elif secs:
        secs[-1].append(l)
sec = secs[which]
rows = list(csv.reader(sec[1:]))
hdr = rows[0]
data = rows[1:]
ie = hdr.index('Instructions Executed')
ss = hdr.index('Warp Stall Sampling (All Samples)')
tot_i = sum(int(r[ie]) for r in data if r[ie].isdigit())
tot_s = sum(int(r[ss]) for r in data if r[ss].isdigit())
print(sec[0][:100], 'instr', tot_i, 'samples', tot_s)
mode = sys.argv[4] if len(sys.argv) > 4 else 'seq'
if mode == 'seq':
    for r in data:
        i = int(r[ie]) if r[ie].isdigit() else 0
        s = int(r[ss]) if r[ss].isdigit() else 0
        if i >= tot_i * 0.002 or s >= tot_s * 0.01:
            print(f'{i:>9} {s:>5}  {r[1][:90]}')
else:
    top = sorted(data, key=lambda r: -(int(r[ss]) if r[ss].isdigit() else 0))[:ntop]
    for r in top:
        print(f'{r[ie]:>9} {r[ss]:>5}  {r[1][:90]}')
