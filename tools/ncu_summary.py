"""Summarise an ncu --set full report: key metrics per kernel + SASS opcode mix.

    python tools/ncu_summary.py report.ncu-rep
"""
import csv, sys, subprocess, collections
rep = sys.argv[1]
out = subprocess.run(["ncu","-i",rep,"--page","details","--csv"],capture_output=True,text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
want = ["DRAM Throughput","Duration","Elapsed Cycles","SM Frequency","Compute (SM) Throughput","Memory Throughput","DRAM Throughput","Issue Slots Busy","Executed Ipc Active","Registers Per Thread","Achieved Occupancy","Theoretical Occupancy","Warp Cycles Per Issued Instruction","Avg. Active Threads Per Warp","Executed Instructions","L1/TEX Hit Rate","L2 Hit Rate","Dynamic Shared Memory Per Block","Block Limit Registers","Block Limit Shared Mem"]
for row in r[1:]:
    name=row[h.index('Metric Name')]
    if name in want:
        print(f"{row[h.index('Kernel Name')][:30]:30s} {name:40s} {row[h.index('Metric Value')]:>14s} {row[h.index('Metric Unit')]}")
out = subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source=sass"],capture_output=True,text=True).stdout
rows=list(csv.reader(out.splitlines()))
hi=[i for i,x in enumerate(rows) if 'Address' in x][0]
h=rows[hi]; data=rows[hi+1:]
isrc=h.index('Source'); iex=h.index('Instructions Executed'); ist=h.index('Warp Stall Sampling (All Samples)')
tot=sum(float(x[iex] or 0) for x in data); stall=sum(float(x[ist] or 0) for x in data)
op=collections.Counter(); st=collections.Counter()
for x in data:
    if len(x)<=max(isrc,iex,ist): continue
    e=float(x[iex] or 0); s=float(x[ist] or 0)
    toks=x[isrc].split()
    if not toks: continue
    o=toks[1] if toks[0].startswith('@') else toks[0]
    o=o.split('.')[0]
    op[o]+=e; st[o]+=s
print('total instr', tot)
fp64=sum(op[k] for k in ('DFMA','DMUL','DADD','DSETP','DMNMX'))
print('FP64 share %.1f%%'%(100*fp64/tot))
for o,e in op.most_common(22): print(f'  {o:10s} {e/tot*100:6.2f}% instr  {st[o]/stall*100:6.2f}% stall')
