"""Aggregate an ncu --page source --print-source sass CSV: instructions executed per opcode and hot spots."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
agg = defaultdict(lambda: [0, 0, 0])
lines = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    ie = int(r[ix["Instructions Executed"]] or 0)
    st = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    agg[op][0] += ie
    agg[op][1] += st
    lines.append((st, ie, r[ix["Address"]], src))
tot = sum(v[0] for v in agg.values())
tst = sum(v[1] for v in agg.values())
print(f"total warp-instr {tot}  stall samples {tst}")
for op, (ie, st, _) in sorted(agg.items(), key=lambda x: -x[1][0])[:30]:
    print(f"{op:12s} {ie:12d} {100*ie/tot:5.1f}%  stall {100*st/max(tst,1):5.1f}%")
print("--- top stall lines")
for st, ie, addr, src in sorted(lines, reverse=True)[:25]:
    print(f"{st:7d} {ie:10d} {addr[-5:]} {src[:80]}")
