"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum
--csv): `python profiles/ncu_launch_summary.py launches.csv [title]`."""
import csv
import sys
from collections import defaultdict


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    tot = defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        if len(r) == len(h) and r[mi] == "gpu__time_duration.sum":
            name = r[ki].split("(")[0]
            tot[name][0] += 1
            tot[name][1] += float(r[vi].replace(",", "")) / 1e3
    allt = sum(v[1] for v in tot.values())
    n = sum(v[0] for v in tot.values())
    if len(sys.argv) > 2:
        print(sys.argv[2])
    print(f"{n} launches, {allt:.1f} us total (serialised, cold cache)")
    for name, (c, t) in sorted(tot.items(), key=lambda x: -x[1][1])[:40]:
        print(f"{name[:60]:60s} n={c:5d} {t:10.1f} us {100 * t / allt:5.1f}%")


if __name__ == "__main__":
    main()
