import csv, sys, collections, subprocess
rep=sys.argv[1]
out=subprocess.run(["ncu","-i",rep,"--page","details","--csv"],capture_output=True,text=True).stdout
rows=list(csv.reader(out.splitlines()))
hdr=rows[0]
want=["Duration","Compute (SM) Throughput","Executed Ipc Active","Issue Slots Busy","Registers Per Thread","Achieved Occupancy","Theoretical Occupancy","Warp Cycles Per Issued Instruction","Avg. Active Threads Per Warp","Executed Instructions","DRAM Throughput","L1/TEX Hit Rate","Eligible Warps Per Scheduler","No Eligible"]
for r in rows[1:]:
    d=dict(zip(hdr,r))
    if d.get("Metric Name") in want: print(f"{d['Metric Name']:40s} {d['Metric Value']} {d['Metric Unit']}")
out=subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source","sass"],capture_output=True,text=True).stdout
rows=list(csv.reader(out.splitlines()))
hdr=rows[1]; data=rows[2:]
ix={h:i for i,h in enumerate(hdr)}
stall_cols=[h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
tot=collections.Counter(); ops=collections.Counter(); ninst=0
for r in data:
    if len(r)<len(hdr): continue
    src=r[ix['Source']].strip().split()
    if not src: continue
    op=src[1] if src[0].startswith('@') else src[0]
    op=op.split('.')[0]
    ex=int(r[ix['Instructions Executed']] or 0); ops[op]+=ex; ninst+=ex
    for c in stall_cols: tot[c]+=int(r[ix[c]] or 0)
print("warp instructions", ninst)
print("ops:", ", ".join(f"{k} {v/ninst*100:.1f}%" for k,v in ops.most_common(12)))
s=sum(tot.values())
print("stalls:", ", ".join(f"{k[6:]} {v/s*100:.1f}%" for k,v in tot.most_common(10)))
