"""Summarise an ncu capture of the step kernel into profiles/ (committed evidence).

  python tools/ncu_summary.py --rep gpurun_out/prof_r1c.ncu-rep --launches gpurun_out/launches_r1c.csv \
      --bench gpurun_out/bench_full.json --tag r1

Writes profiles/<tag>_k_run.md (metrics, stall reasons, launch shares),
profiles/<tag>_launches.csv (the launch list of the timed region) and
profiles/k_run_dram_bytes_per_update.json (read by bench.py for `traffic`).
"""
import argparse
import csv
import io
import json
import os
import shutil
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__occupancy_limit_registers", "smsp__inst_executed.sum",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg",
    "lts__t_sectors.sum", "lts__t_sectors_srcunit_ltcfabric.sum",
]


def raw(rep):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], stderr=subprocess.DEVNULL).decode()
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--launches", required=True)
    ap.add_argument("--bench", default=None)
    ap.add_argument("--tag", default="r1")
    ap.add_argument("--steady-steps", type=int, default=0,
                    help="the capture is one steady launch of this many steps (no flush): labelled so, per-step "
                         "figures added, k_run_dram_bytes_per_update.json left alone")
    a = ap.parse_args()
    h, u, rows = raw(a.rep)
    v = rows[0]
    m = {n: (v[i], u[i]) for i, n in enumerate(h)}
    stalls = []
    for i, n in enumerate(h):
        if n.startswith("smsp__pcsamp_warps_issue_stalled") and not n.endswith("not_issued"):
            try:
                stalls.append((float(v[i].replace(",", "")), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    tot = sum(x for x, _ in stalls) or 1.0
    dram = (float(m["dram__bytes_read.sum"][0].replace(",", "")) * (1e6 if m["dram__bytes_read.sum"][1] == "Mbyte" else 1e3 if m["dram__bytes_read.sum"][1] == "Kbyte" else 1e9 if m["dram__bytes_read.sum"][1] == "Gbyte" else 1)
            + float(m["dram__bytes_write.sum"][0].replace(",", "")) * (1e6 if m["dram__bytes_write.sum"][1] == "Mbyte" else 1e3 if m["dram__bytes_write.sum"][1] == "Kbyte" else 1e9 if m["dram__bytes_write.sum"][1] == "Gbyte" else 1))
    # launch list
    lrows = list(csv.reader(open(a.launches)))
    hi = [i for i, r in enumerate(lrows) if r and r[0] == "ID"][0]
    lh = lrows[hi]
    ki, vi = lh.index("Kernel Name"), lh.index("Metric Value")
    launches = [(r[ki], float(r[vi].replace(",", ""))) for r in lrows[hi + 1:] if len(r) > vi]
    totl = sum(t for _, t in launches) or 1.0
    agg = {}
    for k, t in launches:
        name = k.split("(")[0].replace("void ", "")[:80]
        agg.setdefault(name, [0, 0.0])
        agg[name][0] += 1
        agg[name][1] += t
    bench = json.load(open(a.bench)) if a.bench and os.path.exists(a.bench) else None
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    shutil.copy(a.launches, os.path.join(ROOT, "profiles", "%s_launches.csv" % a.tag))
    wl = bench["config"]["workload"] if bench else "the bench's"
    if a.steady_steps:
        src = ("Source: `%s` (ncu --set full --clock-control none): one **steady-state** launch of %d simulation "
               "steps in one `lpsim_step` call at the AM peak of the %s workload, **no L2 flush** (bench.py's NVTX "
               "range `steady`, the second k_run launch: the one after the sort).  Per-step figures are the launch's "
               "divided by %d.  The launch table is the cold one-step launch list of the same round (`%s`)."
               % (os.path.basename(a.rep), a.steady_steps, wl, a.steady_steps, os.path.basename(a.launches)))
    else:
        src = ("Source: `%s` (ncu --set full --clock-control none, one timed launch = one simulation step at the AM "
               "peak of the %s workload, L2 flushed before the step), launch list `%s` (ncu --metrics "
               "gpu__time_duration.sum over bench.py's NVTX range `timed`)." % (os.path.basename(a.rep), wl,
                                                                                 os.path.basename(a.launches)))
    md = ["# %s — ncu summary of `k_run` (the fused step kernel)" % a.tag, "", src, "",
          "| metric | value | unit |", "|---|---|---|"]
    for n in WANT:
        if n in m:
            md.append("| %s | %s | %s |" % (n, m[n][0], m[n][1]))
    md += ["| dram bytes per launch (read+write) | %.0f | byte |" % dram]
    if a.steady_steps:
        md += ["| dram bytes per step (read+write) | %.0f | byte |" % (dram / a.steady_steps),
               "| device time per step | %.3f | us |" % (float(m["gpu__time_duration.sum"][0].replace(",", "")) *
                                                        (1e3 if m["gpu__time_duration.sum"][1] == "ms" else 1.0) /
                                                        a.steady_steps)]
    lts = None
    if "lts__t_sectors.sum" in m:  # L2 traffic: sectors x 32 B; the share crossing the fabric between the dies
        lts = 32.0 * float(m["lts__t_sectors.sum"][0].replace(",", ""))
        md.append("| L2 bytes per launch (lts__t_sectors.sum x 32 B) | %.0f | byte |" % lts)
        if "lts__t_sectors_srcunit_ltcfabric.sum" in m:
            fab = 32.0 * float(m["lts__t_sectors_srcunit_ltcfabric.sum"][0].replace(",", ""))
            md.append("| of which from the other die (ltcfabric) | %.0f (%.1f %%) | byte |" % (fab, 100 * fab / lts))
    md.append("")
    md += ["## Warp stall reasons (pc sampling, share)", "", "| reason | share |", "|---|---|"]
    for x, n in stalls[:10]:
        md.append("| %s | %.1f %% |" % (n, 100 * x / tot))
    md += ["", "## Launches in the timed region (cold-cache, serialised)", "", "| kernel | launches | total us | share |",
           "|---|---|---|---|"]
    for name, (cnt, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        md.append("| %s | %d | %.1f | %.1f %% |" % (name, cnt, t / 1e3, 100 * t / totl))
    md.append("")
    upd = None
    if bench:
        w = bench.get("window", {})
        upd = bench["value"] * bench["ms_per_step"] / 1e3  # updates per step
        md += ["## Bench line of the same build", "", "```json", json.dumps(bench, indent=1)[:4000], "```", ""]
        md.append("DRAM bytes per vehicle-update (ncu launch / updates per step from the bench): %.1f B "
                  "(algorithmic: %d B)." % (dram / max(1, a.steady_steps) / upd, bench["roofline"]["alg_bytes_per_update"]))
    open(os.path.join(ROOT, "profiles", "%s_k_run.md" % a.tag), "w").write("\n".join(md) + "\n")
    if a.steady_steps:
        print("\n".join(md))
        return
    json.dump({"tag": a.tag, "dram_bytes_per_launch": dram, "l2_bytes_per_launch": lts, "updates_per_step_bench": upd,
               "dram_bytes_per_update": (dram / upd) if upd else None,
               "kernel_us": float(m["gpu__time_duration.sum"][0].replace(",", "")),
               "source": "profiles/%s_k_run.md (%s, ncu --set full, one cold step)" % (a.tag, os.path.basename(a.rep))},
              open(os.path.join(ROOT, "profiles", "k_run_dram_bytes_per_update.json"), "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
