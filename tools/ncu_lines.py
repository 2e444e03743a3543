"""Per-CUDA-line warp-stall samples of an ncu report (needs -lineinfo + --import-source)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                              stderr=subprocess.DEVNULL).decode()
rows = list(csv.reader(io.StringIO(out)))
res = []
cur = None
for r in rows:
    if len(r) > 5 and r[0] not in ("", "Line No") and r[0].isdigit():
        try:
            res.append((int(r[4]), int(r[0]), r[1][:100]))
        except ValueError:
            pass
tot = sum(x for x, _, _ in res) or 1
for x, ln, src in sorted(res, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print("%5.1f%%  L%-5d %s" % (100.0 * x / tot, ln, src))
