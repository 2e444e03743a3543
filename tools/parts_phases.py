"""Phase times (LPSIM_FLAG_TIMING, instrumented kernel) of the K-partition step at the AM peak, one
process on one GPU, partitions balanced for the peak's load (multi.pilot_partition): where the K > 1
step spends its time relative to K = 1.

usage: python tools/parts_phases.py [workload] [--ks 1,2,4,8] [--steps 128]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2406_08496_b200 import FLAG_TIMING, Simulation  # noqa: E402
from paper_2406_08496_b200.multi import pilot_partition  # noqa: E402
from workloads import make_workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload", nargs="?", default="bay9m")
ap.add_argument("--ks", default="1,2,4,8")
ap.add_argument("--peak-s", type=float, default=8 * 3600.0)
ap.add_argument("--steps", type=int, default=128)
args = ap.parse_args()

g, d, meta = make_workload(args.workload, cache_dir="/tmp/lpsim_cache")
for k in [int(x) for x in args.ks.split(",")]:
    kw = {}
    if k > 1:
        part = pilot_partition(g, d, k, args.peak_s)
        kw = dict(num_parts=k, node_part=part.ctypes.data)
    for flags, label in ((0, "lean"), (FLAG_TIMING, "timing")):
        sim = Simulation(g, flags=0, **kw)
        sim.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
        sim.step(int(args.peak_s / 0.5))
        sim.set_flags(flags)
        sim.step(args.steps)
        st = sim.stats()
        n = args.steps
        row = {"k": k, "kernel": label, "us_per_step": round(1e3 * st["step_ms"] / n, 2),
               "sort_us_per_step": round(1e3 * st.get("sort_ns", 0) / 1e6 / n, 3), "on_road": st["on_road"]}
        if flags:
            row["phase_us_per_step"] = [round(x / 1e3 / n, 2) for x in st["phase_ns"]]
        print(json.dumps(row), flush=True)
        sim.close()
