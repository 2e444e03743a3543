"""Per-step device time over a full-demand run (the bench's full_run): chunks of 1,800 steps (15 min),
vehicles on the road at each chunk's end, device us per step.  Shows where the full run's device
time goes (peak vs the light-load head and drain tail).

usage: python tools/day_profile.py [workload] [--grid N]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2406_08496_b200 import Simulation  # noqa: E402
from workloads import make_workload  # noqa: E402

g, d, meta = make_workload(sys.argv[1] if len(sys.argv) > 1 else "bay9m", cache_dir="/tmp/lpsim_cache")
sim = Simulation(g)
sim.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
steps, dev = 0, 0.0
rows = []
while True:
    sim.step(1800)
    steps += 1800
    st = sim.stats()
    dev += st["step_ms"]
    rows.append({"step": steps, "on_road": st["on_road"], "us_per_step": round(1e3 * st["step_ms"] / 1800, 2),
                 "arrived": st["arrivals"]})
    print(json.dumps(rows[-1]), flush=True)
    if steps >= meta["horizon_s"] / 0.5 and st["arrivals"] == meta["trips"]:
        break
    if steps >= 2 * meta["horizon_s"] / 0.5:
        break
print(json.dumps({"total_device_s": dev / 1e3, "steps": steps}), flush=True)
