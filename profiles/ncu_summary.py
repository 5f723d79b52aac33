"""Summarise an ncu report (read here, no GPU needed):

  python profiles/ncu_summary.py gpurun_out/prof.ncu-rep [kernel-regex]

Prints per launch: duration, DRAM bytes read/written, DRAM throughput %,
achieved occupancy, registers, L2 hit rate and the top warp stall reasons.
"""

import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

RAW = {
    "gpu__time_duration.sum": "time",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occ_pct",
    "launch__registers_per_thread": "regs",
    "lts__t_sector_hit_rate.pct": "l2_hit",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__cycles_active.avg": "cyc",
}


PEAK = 6546.9  # GB/s, MEASURED_PEAKS.json copy bandwidth on this pool's B200s
_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
          "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
          "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def achieved(hdr, units, r):
    """(dram read + write bytes) / duration in GB/s, or None."""
    try:
        b = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(k)
            b += float(r[i].replace(",", "")) * _SCALE[units[i]]
        i = hdr.index("gpu__time_duration.sum")
        t = float(r[i].replace(",", "")) * _SCALE[units[i]]
        return b / t / 1e9 if t > 0 else None
    except (ValueError, KeyError):
        return None


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(out.stdout)))
    return rows[0], rows[1], rows[2:]


def main():
    rep = sys.argv[1]
    pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
    hdr, units, rows = raw_rows(rep)
    stall_cols = [i for i, h in enumerate(hdr)
                  if h.startswith("smsp__average_warp_latency_issue_stalled_")
                  or h.startswith("smsp__pcsamp_warps_issue_stalled_")]
    for r in rows:
        name = r[hdr.index("Kernel Name")]
        if pat and not pat.search(name):
            continue
        vals = {}
        for k, short in RAW.items():
            if k in hdr:
                i = hdr.index(k)
                vals[short] = f"{r[i]} {units[i]}".strip()
        stalls = []
        for i in stall_cols:
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            stalls.append((v, hdr[i].split("stalled_")[-1]))
        stalls.sort(reverse=True)
        print(name[:90])
        print("   " + "  ".join(f"{k}={v}" for k, v in vals.items()))
        bw = achieved(hdr, units, r)
        if bw is not None:
            print(f"   achieved DRAM {bw:.0f} GB/s = {bw / PEAK:.2f} of the measured "
                  f"{PEAK:.0f} GB/s copy peak")
        if stalls:
            print("   stalls: " + ", ".join(f"{n}={v:.3g}" for v, n in stalls[:6]))


if __name__ == "__main__":
    main()
