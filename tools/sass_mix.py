"""Aggregate an ncu --page source --csv (SASS view) by opcode: executed warp
instructions and stall samples.  usage: sass_mix.py source_<kernel>.csv"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
i = next(k for k, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[i]
ix = hdr.index("Source"); ie = hdr.index("Instructions Executed"); isamp = hdr.index("Warp Stall Sampling (All Samples)")
cnt = collections.Counter(); smp = collections.Counter()
tot = 0; tots = 0
for r in rows[i + 1:]:
    if len(r) <= ie or not r[ie]:
        continue
    op = r[ix].split()[0] if r[ix].split() else "?"
    if op.startswith("@"):
        op = r[ix].split()[1]
    op = op.split(".")[0]
    n = float(r[ie] or 0); s = float(r[isamp] or 0)
    cnt[op] += n; smp[op] += s; tot += n; tots += s
print(f"total warp insts {tot:.0f}  samples {tots:.0f}")
for op, n in cnt.most_common(30):
    print(f"{op:10s} {n:12.0f} {100*n/tot:5.1f}%  stall-samples {100*smp[op]/max(tots,1):5.1f}%")
