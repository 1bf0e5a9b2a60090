"""Stall reasons of an ncu source-page CSV (--page source --csv --print-source sass) split into
address regions: python tools/ncu_regions.py <src.csv> <hexaddr_lo>:<hexaddr_hi>[:name] ..."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
iA, iE, iS = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Source")
st = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
for spec in sys.argv[2:]:
    parts = spec.split(":")
    lo, hi = int(parts[0], 16), int(parts[1], 16)
    name = parts[2] if len(parts) > 2 else spec
    sel = [r for r in data if lo <= int(r[iA], 16) < hi]
    c = collections.Counter()
    for r in sel:
        for i in st:
            c[hdr[i][6:]] += int(r[i] or 0)
    tot = sum(c.values()) or 1
    ins = sum(int(r[iE] or 0) for r in sel)
    ops = collections.Counter()
    for r in sel:
        op = r[iS].strip().split()
        op = [o for o in op if not o.startswith("@")]
        if op: ops[op[0].split(".")[0]] += int(r[iE] or 0)
    print(f"{name}: {len(sel)} sass, {ins} warp-instrs, {tot} samples: " +
          ", ".join(f"{k} {100*v/tot:.0f}%" for k, v in c.most_common(8)))
    print("   mix: " + ", ".join(f"{k} {v}" for k, v in ops.most_common(12)))
