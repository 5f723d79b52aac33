"""Per-kernel summary of an ncu CSV capture with DRAM metrics
(profiles/ncu_all.sh): launches, total and mean duration, share of the step,
DRAM bytes per launch, achieved DRAM GB/s and its fraction of the measured
copy peak, L2 hit rate, occupancy, registers, grid.

    python profiles/ncu_all_summary.py all_c2.csv[.gz] [title]
"""
import csv
import gzip
import io
import sys
from collections import defaultdict

PEAK = 6546.9  # GB/s, MEASURED_PEAKS.json copy bandwidth (B200 pool)
_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9,
          "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "%": 1.0, "": 1.0,
          "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
          "register/thread": 1.0}


def rows(path):
    op = gzip.open if path.endswith(".gz") else open
    with op(path, "rt") as f:
        text = f.read()
    lines = text.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    return list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))


def main():
    data = rows(sys.argv[1])
    per = defaultdict(dict)  # launch id -> metrics
    for r in data:
        d = per[r["ID"]]
        d["name"] = r["Kernel Name"]
        try:
            v = float(r["Metric Value"].replace(",", ""))
        except ValueError:
            continue
        d[r["Metric Name"]] = v * _SCALE.get(r.get("Metric Unit", ""), 1.0)
    agg = defaultdict(lambda: defaultdict(float))
    for d in per.values():
        name = d["name"].split("(")[0]
        if name.startswith("void "):
            name = name[5:]
        a = agg[name]
        a["n"] += 1
        a["t"] += d.get("gpu__time_duration.sum", 0.0)
        a["b"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        a["l2"] += d.get("lts__t_sector_hit_rate.pct", 0.0)
        a["occ"] += d.get("sm__warps_active.avg.pct_of_peak_sustained_active", 0.0)
        a["regs"] = d.get("launch__registers_per_thread", 0.0)
        a["grid"] = max(a["grid"], d.get("launch__grid_size", 0.0))
    tot = sum(a["t"] for a in agg.values())
    if len(sys.argv) > 2:
        print(sys.argv[2])
    print(f"{sum(int(a['n']) for a in agg.values())} launches, {tot * 1e6:.1f} us total "
          "(serialised, cold cache); peak = measured copy bandwidth "
          f"{PEAK} GB/s")
    print(f"{'kernel':58s} {'n':>5s} {'share':>6s} {'us/launch':>9s} {'MB/launch':>9s} "
          f"{'DRAM GB/s':>9s} {'frac':>5s} {'L2hit':>5s} {'occ':>4s} {'regs':>4s} {'grid':>6s}")
    for name, a in sorted(agg.items(), key=lambda x: -x[1]["t"]):
        n = a["n"]
        gbs = a["b"] / a["t"] / 1e9 if a["t"] else 0.0
        print(f"{name[:58]:58s} {int(n):5d} {100 * a['t'] / tot:5.1f}% {a['t'] / n * 1e6:9.2f} "
              f"{a['b'] / n / 1e6:9.2f} {gbs:9.0f} {gbs / PEAK:5.2f} {a['l2'] / n:5.1f} "
              f"{a['occ'] / n:4.0f} {int(a['regs']):4d} {int(a['grid']):6d}")


if __name__ == "__main__":
    main()
