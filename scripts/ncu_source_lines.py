"""Per-CUDA-source-line executed warp instructions of one kernel in an ncu report
(--page source, cuda,sass): python scripts/ncu_source_lines.py rep.ncu-rep <kernel regex> [top] [column],
column e.g. "Warp Stall Sampling (All Samples)" instead of "Instructions Executed"."""
import csv, collections, sys, subprocess
rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu","-i",rep,"--page","source","--csv","--kernel-name","regex:"+kern,"--print-source","cuda,sass"],capture_output=True,text=True).stdout
rows=list(csv.reader(out.splitlines()))
hdr=[r for r in rows if r and r[0]=='Line No'][0]
i_ex=hdr.index(sys.argv[4] if len(sys.argv)>4 else "Instructions Executed")
res=collections.Counter(); src={}
f=None
for r in rows:
    if len(r)<3: 
        if r and r[0]=='File Path': f=r[1].split('/')[-1]
        continue
    if r[0] in ('File Path',): f=r[1].split('/')[-1]; continue
    if r[0] in ('Line No','Function Name'): continue
    if r[0]!='':
        try: ex=float(r[i_ex] or 0)
        except: ex=0
        res[(f,r[0])]+=ex; src[(f,r[0])]=r[1][:80]
tot=sum(res.values())
print("total", tot)
for k,e in res.most_common(int(sys.argv[3]) if len(sys.argv)>3 else 25): print(f"{e/tot*100:5.1f}% {e:12.0f} {k[0]}:{k[1]} {src[k]}")
