"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum launch list:
python tools/launch_summary.py launches.csv"""

import csv
import re
import sys
from collections import OrderedDict


def main(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    agg = OrderedDict()
    seq = []
    for r in rows[hdr + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[ki])[:70]
        t = float(r[vi].replace(",", ""))
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += t
        seq.append((name, t))
    for name, t in seq:
        print(f"{t / 1e3:10.1f} us  {name}")
    print("---")
    for name, (n, t) in agg.items():
        print(f"{n:5d} x {t / n / 1e3:9.1f} us  {name}")


if __name__ == "__main__":
    main(sys.argv[1])
