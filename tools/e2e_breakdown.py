"""Where the end-to-end wall time of a full-demand run goes (the bench's `e2e` / `full_run`): create,
load_demand, the step calls (wall vs device), results.

usage: python tools/e2e_breakdown.py [workload]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2406_08496_b200 import Simulation  # noqa: E402
from workloads import make_workload  # noqa: E402

g, d, meta = make_workload(sys.argv[1] if len(sys.argv) > 1 else "bay9m", cache_dir="/tmp/lpsim_cache")
for rep in range(2):
    t = {}
    t0 = time.perf_counter()
    sim = Simulation(g)
    t["create"] = time.perf_counter() - t0
    t1 = time.perf_counter()
    sim.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
    t["load_demand"] = time.perf_counter() - t1
    t2 = time.perf_counter()
    steps, dev, stats_s = 0, 0.0, 0.0
    while True:
        sim.step(3600)
        steps += 3600
        ts = time.perf_counter()
        st = sim.stats()
        stats_s += time.perf_counter() - ts
        dev += st["step_ms"] / 1e3
        if steps >= meta["horizon_s"] / 0.5 and st["arrivals"] == meta["trips"]:
            break
    t["step_calls_wall"] = time.perf_counter() - t2
    t["step_calls_device"] = dev
    t["stats_calls"] = stats_s
    t3 = time.perf_counter()
    a, tt, dist = sim.results()
    t["results"] = time.perf_counter() - t3
    t["total"] = time.perf_counter() - t0
    t["steps"] = steps
    sim.close()
    print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in t.items()}), flush=True)
