"""Instructions executed and warp-stall samples per CUDA source line of one ncu report.

usage: python tools/ncu_lines.py REPORT.ncu-rep [TOP] [FIRST_LINE LAST_LINE]
SASS rows are attributed to the preceding source row (ncu --page source --print-source cuda,sass).
An optional line range restricts the table (e.g. one phase of the step kernel).
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
lo, hi = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (0, 1 << 30)
out = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                              stderr=subprocess.DEVNULL).decode()
hdr = None
cur = None
fname = None
src, ie, ss = {}, collections.Counter(), collections.Counter()
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Name":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        iei, ssi = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if not hdr or len(r) < len(hdr):
        continue
    if r[0].isdigit():
        cur = (fname, int(r[0]))
        src[cur] = r[1][:100]
        continue
    if r[0] == "" and cur is not None:
        try:
            ie[cur] += int(r[iei] or 0)
            ss[cur] += int(r[ssi] or 0)
        except ValueError:
            pass
tie, tss = sum(ie.values()) or 1, sum(ss.values()) or 1
sel = [k for k in src if lo <= k[1] <= hi and k[0] == "lpsim_step.cu"] if len(sys.argv) > 4 else list(src)
print("total: %d warp-instructions, %d stall samples; selection: %.1f%% inst, %.1f%% samples" % (
    tie, tss, 100 * sum(ie[k] for k in sel) / tie, 100 * sum(ss[k] for k in sel) / tss))
print(" inst%  stall%  line")
for k in sorted(sel, key=lambda k: -(ss[k] + ie[k] * tss / tie))[:top]:
    print("%6.2f %6.2f  %s:%d  %s" % (100 * ie[k] / tie, 100 * ss[k] / tss, k[0], k[1], src[k]))
