"""Group an ncu SASS source-page CSV into straight-line runs of equal execution count."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.004
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
blocks, cur = [], None
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    ie = int(r[ix["Instructions Executed"]] or 0)
    st = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    src = r[ix["Source"]]
    if cur and cur[0] == ie:
        cur[1] += 1
        cur[2] += st
        cur[3].append(src)
    else:
        cur = [ie, 1, st, [src]]
        blocks.append(cur)
tot = sum(b[0] * b[1] for b in blocks)
tst = sum(b[2] for b in blocks)
print("total warp-instr", tot, "stall samples", tst)
for b in blocks:
    if b[0] * b[1] > thr * tot or b[2] > thr * tst:
        print(f"{b[0]:9d} x{b[1]:4d} = {b[0]*b[1]/tot*100:5.1f}%  stall {100*b[2]/tst:5.1f}%  {b[3][0][:45]} ... {b[3][-1][:40]}")
