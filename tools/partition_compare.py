"""Partitioner comparison (§8(f) item 1): cut lanes (= migrant slots + entry-halo lanes, the static
exchange shape), the largest part's share of the route-visit weight, and host time, for the
route-weighted RCB, the balanced multilevel k-way partition (the built-in one), the unbalanced
Leiden + k-means partition and a random partition, on one workload.  With --steps, also the single-GPU multi-partition step time of each
(one process, K partitions, in-kernel exchange) at the window the bench uses.

usage: python tools/partition_compare.py [workload] [--ks 2,4,8] [--steps N]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2406_08496_b200.lpsim import (lpsim_partition_leiden_kmeans, lpsim_partition_multilevel,  # noqa: E402
                                         lpsim_partition_rcb, lpsim_plan_cut_lanes)
from paper_2406_08496_b200.multi import route_weights  # noqa: E402
from workloads import make_workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload", nargs="?", default="bay9m")
ap.add_argument("--ks", default="2,4,8")
ap.add_argument("--steps", type=int, default=0)
ap.add_argument("--peak-s", type=float, default=8 * 3600.0)
ap.add_argument("--window-s", type=float, default=0.0, help="time-windowed weights: only trips departing in "
                "[peak-s - window-s, peak-s] count (0 = the whole day)")
args = ap.parse_args()

g, d, meta = make_workload(args.workload, cache_dir="/tmp/lpsim_cache")
n = g["row_ptr"].shape[0] - 1
dw = d
if args.window_s > 0:  # route visits of the trips departing in the window only
    keep = (d["depart_s"] >= args.peak_s - args.window_s) & (d["depart_s"] < args.peak_s)
    idx = np.nonzero(keep)[0]
    lens = d["route_ptr"][idx + 1] - d["route_ptr"][idx]
    rp = np.zeros(idx.size + 1, np.int64)
    np.cumsum(lens, out=rp[1:])
    re = np.concatenate([d["route_edges"][d["route_ptr"][i]:d["route_ptr"][i + 1]] for i in idx]) if idx.size else \
        np.zeros(0, np.int32)
    dw = {"depart_s": d["depart_s"][idx], "route_ptr": rp, "route_edges": re}
w = route_weights(g, dw).astype(np.float64)
rows = []
for k in [int(x) for x in args.ks.split(",")]:
    rng = np.random.default_rng(k)
    parts = {}
    t0 = time.perf_counter(); parts["rcb"] = lpsim_partition_rcb(n, g.get("node_xy"), w, k); t1 = time.perf_counter()
    parts["multilevel"] = lpsim_partition_multilevel(g, k, node_weight=w, imbalance=0.05, seed=1)
    t2 = time.perf_counter()
    parts["leiden_kmeans"] = lpsim_partition_leiden_kmeans(g, k, node_weight=w, seed=1)
    t3 = time.perf_counter()
    parts["random"] = rng.integers(0, k, n).astype(np.int32)
    host = {"rcb": t1 - t0, "multilevel": t2 - t1, "leiden_kmeans": t3 - t2, "random": 0.0}
    for name, p in parts.items():
        cut = int(lpsim_plan_cut_lanes(g, p, k).sum())
        loads = np.bincount(p, weights=w, minlength=k)
        row = {"workload": args.workload, "k": k, "partition": name, "cut_lanes": cut,
               "max_part_share": round(float(loads.max() / max(w.sum(), 1e-12)), 4),
               "balance": round(float(loads.max() / max(loads.mean(), 1e-12)), 4),
               "host_s": round(host[name], 3)}
        if args.steps:
            from paper_2406_08496_b200 import Simulation
            sim = Simulation(g, num_parts=k, node_part=p.ctypes.data, flags=0)
            sim.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
            sim.step(int(args.peak_s / 0.5))
            sim.step(args.steps)
            st = sim.stats()
            row.update(us_per_step=round(1e3 * st["step_ms"] / args.steps, 2),
                       exchange_us_per_step=round(1e3 * st["exchange_ms"] / args.steps, 2), on_road=st["on_road"])
            sim.close()
        rows.append(row)
        print(json.dumps(row), flush=True)
