"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import csv
import sys
from collections import OrderedDict


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
    out = []
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        out.append((int(r[ii]), r[ki].split("(")[0], float(r[vi].replace(",", ""))))
    return out


if __name__ == "__main__":
    seq = load(sys.argv[1])
    if len(sys.argv) > 2:
        for s in seq[: int(sys.argv[2])]:
            print(s)
    agg = OrderedDict()
    for _, n, v in seq:
        a = agg.setdefault(n, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    for n, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{v / tot * 100:6.2f}%  {c:4d} launches  {v / c / 1e3:10.1f} us/launch  {n}")
