"""Warp-stall samples per CUDA source line (SASS rows attributed to the preceding source row)."""
import csv, io, subprocess, sys
from collections import defaultdict
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                              stderr=subprocess.DEVNULL).decode()
rows = list(csv.reader(io.StringIO(out)))
hdr = None
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        break
si = hdr.index("Warp Stall Sampling (All Samples)")
agg = defaultdict(int)
src = {}
cur = None
for r in rows:
    if len(r) <= si:
        continue
    if r[0].isdigit():
        cur = int(r[0])
        src[cur] = r[1][:110]
        continue
    if r[0] == "" and cur is not None:
        try:
            agg[cur] += int(r[si])
        except ValueError:
            pass
tot = sum(agg.values()) or 1
for ln, x in sorted(agg.items(), key=lambda t: -t[1])[:top]:
    print("%5.1f%%  L%-5d %s" % (100.0 * x / tot, ln, src.get(ln, "")))
