import csv, subprocess, sys
rep, which = sys.argv[1], int(sys.argv[2])
thr = int(sys.argv[3]) if len(sys.argv) > 3 else 150000
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
secs=[]
for l in out.splitlines():
    if l.startswith('"Kernel Name"'): secs.append([l])
    elif secs: secs[-1].append(l)
print(len(secs), 'sections')
sec=secs[which]
print(sec[0][:110])
rows=list(csv.reader(sec[1:])); hdr=rows[0]; data=rows[1:]
ie=hdr.index('Instructions Executed'); ss=hdr.index('Warp Stall Sampling (All Samples)')
blocks=[]
for r in data:
    c=int(r[ie]) if r[ie].isdigit() else 0
    s=int(r[ss]) if r[ss].isdigit() else 0
    if blocks and blocks[-1][0]==c: blocks[-1][1]+=1; blocks[-1][2].append(r[1].strip()[:45]); blocks[-1][3]+=s
    else: blocks.append([c,1,[r[1].strip()[:45]],s])
tot=0; tots=0
for c,n,ins,s in blocks:
    tot+=c*n; tots+=s
for c,n,ins,s in blocks:
    if c*n>thr or s>tots*0.02: print(f"{c:>8} x{n:>4} = {c*n:>9} stall={s:>5}  {ins[0]} ... {ins[-1]}")
print('total',tot,'samples',tots)
