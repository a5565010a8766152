"""Per-source-line instruction / stall shares of an ncu report (needs -lineinfo).

    python tools/ncu_lines.py report.ncu-rep [top]
"""
import csv, sys, subprocess, collections
rep=sys.argv[1]; top=int(sys.argv[2]) if len(sys.argv)>2 else 40
out=subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source=cuda,sass"],capture_output=True,text=True).stdout
rows=list(csv.reader(out.splitlines()))
hi=[i for i,x in enumerate(rows) if x and x[0]=='Line No'][0]
h=rows[hi]
iex=h.index('Instructions Executed'); ist=h.index('Warp Stall Sampling (All Samples)')
line_instr=collections.Counter(); line_stall=collections.Counter(); src={}
cur=None
for x in rows[hi+1:]:
    if len(x)<=iex: continue
    if x[0]:
        if not x[0].isdigit():
            continue
        cur=int(x[0]); src[cur]=x[1]
    try:
        e=float(x[iex] or 0); s=float(x[ist] or 0)
    except ValueError: continue
    line_instr[cur]+=e; line_stall[cur]+=s
tot=sum(line_instr.values()); ts=sum(line_stall.values())
print('total', tot)
for ln,e in sorted(line_instr.items(), key=lambda kv:-kv[1])[:top]:
    print(f"{ln:5d} {100*e/tot:6.2f}% instr {100*line_stall[ln]/ts:6.2f}% stall | {src.get(ln,'')[:90]}")
