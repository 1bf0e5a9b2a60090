import csv,sys,collections,re
rows=list(csv.reader(open(sys.argv[1])))
hdr=rows[1]; data=rows[2:]
iE=hdr.index("Instructions Executed"); iS=hdr.index("Source"); iW=hdr.index("Warp Stall Sampling (All Samples)")
tot=sum(int(r[iE] or 0) for r in data); totw=sum(int(r[iW] or 0) for r in data)
print("total warp instrs",tot, "samples", totw)
c=collections.Counter(); s=collections.Counter()
for r in data:
    op=re.sub(r'^@!?U?P\w+\s+','',r[iS].strip()).split()[0] if r[iS].strip() else '?'
    base=op.split('.')[0]
    c[base]+=int(r[iE] or 0); s[base]+=int(r[iW] or 0)
for k,v in c.most_common(30): print(f"{k:10s} {v/tot*100:6.1f}% instr  {s[k]/totw*100:6.1f}% stall-samples")
