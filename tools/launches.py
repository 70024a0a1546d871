"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel name."""
import csv
import sys
from collections import defaultdict


def main(path, skip_names=()):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(r for r in rows if r[0] == "ID")
    agg = defaultdict(lambda: [0, 0.0])
    seq = []
    for r in rows:
        if r[0] == "ID" or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        name = d["Kernel Name"]
        t = float(d["Metric Value"].replace(",", ""))
        agg[name][0] += 1
        agg[name][1] += t
        seq.append((name, t))
    tot = sum(v[1] for v in agg.values())
    for name, (cnt, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{cnt:4d} {t / 1e3:10.1f} us {100 * t / tot:5.1f}%  {name[:90]}")
    return seq


if __name__ == "__main__":
    seq = main(sys.argv[1])
    if len(sys.argv) > 2:
        print("--- last", sys.argv[2], "launches")
        for name, t in seq[-int(sys.argv[2]):]:
            print(f"{t / 1e3:9.1f} us  {name[:90]}")
