"""Top SASS instructions by warp-stall samples from an ncu report:
  python profiles/ncu_hotspots.py rep.ncu-rep [kernel-regex] [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"]
if len(sys.argv) > 2:
    args += ["-k", "regex:" + sys.argv[2]]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
rows = list(csv.reader(io.StringIO(subprocess.run(args, capture_output=True, text=True).stdout)))
hi = next(i for i, r in enumerate(rows) if "Source" in r and "Address" in r)
hdr = rows[hi]
si, ai = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
data = []
for r in rows[hi + 1:]:
    if len(r) <= ai:
        continue
    try:
        v = float(r[ai])
    except ValueError:
        continue
    top = sorted(((float(r[i] or 0), hdr[i][6:]) for i in stall_cols), reverse=True)[:2]
    data.append((v, r[hdr.index("Address")], r[si], top))
tot = sum(d[0] for d in data) or 1
for v, addr, src, top in sorted(data, reverse=True)[:n]:
    print(f"{100 * v / tot:5.1f}% {addr:>6} {src[:70]:70s} {top}")
