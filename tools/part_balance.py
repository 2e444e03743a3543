"""Per-partition load at the AM peak (vehicles on the road whose edge each part owns) for the
route-weighted multilevel partition (§8(e)) with node weights = route visits of the whole
day (the built-in partition) or of the trips departing in a window before the peak; and, with
--steps, the K-partition step at the peak in one process on one GPU for each.

usage: python tools/part_balance.py [workload] [--ks 2,4,8] [--windows 0,3600,7200] [--steps 128]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2406_08496_b200 import Simulation  # noqa: E402
from paper_2406_08496_b200.lpsim import lpsim_partition_multilevel, lpsim_plan_cut_lanes  # noqa: E402
from paper_2406_08496_b200.multi import route_weights  # noqa: E402
from workloads import make_workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload", nargs="?", default="bay9m")
ap.add_argument("--ks", default="2,4,8")
ap.add_argument("--windows", default="0,3600,7200",
                help="node weights: route visits of the trips departing in [peak - w, peak) (0 = whole day); "
                     "-1 = vehicles on the node's in-edges at the peak (a pilot run's occupancy)")
ap.add_argument("--peak-s", type=float, default=8 * 3600.0)
ap.add_argument("--steps", type=int, default=0)
args = ap.parse_args()

g, d, meta = make_workload(args.workload, cache_dir="/tmp/lpsim_cache")
n = g["row_ptr"].shape[0] - 1
col = np.asarray(g["dst"])  # destination node of each edge

sim = Simulation(g, flags=0)
sim.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
sim.step(int(args.peak_s / 0.5))
ts = sim.trip_state()
sim.close()
on = ts["status"] == 1
e_on = ts["edge"][on]
print(json.dumps({"on_road": int(on.sum())}), flush=True)


def window_demand(win):
    if win <= 0:
        return d
    keep = (d["depart_s"] >= args.peak_s - win) & (d["depart_s"] < args.peak_s)
    idx = np.nonzero(keep)[0]
    lens = d["route_ptr"][idx + 1] - d["route_ptr"][idx]
    rp = np.zeros(idx.size + 1, np.int64)
    np.cumsum(lens, out=rp[1:])
    re = np.concatenate([d["route_edges"][d["route_ptr"][i]:d["route_ptr"][i + 1]] for i in idx])
    return {"depart_s": d["depart_s"][idx], "route_ptr": rp, "route_edges": re}


for k in [int(x) for x in args.ks.split(",")]:
    for win in [float(x) for x in args.windows.split(",")]:
        if win < 0:
            w = np.bincount(col[e_on], minlength=n).astype(np.float64)
        else:
            w = route_weights(g, window_demand(win)).astype(np.float64)
        p = lpsim_partition_multilevel(g, k, node_weight=w, imbalance=0.03, seed=1)
        loads = np.bincount(p[col[e_on]], minlength=k)
        row = {"k": k, "window_s": win, "cut_lanes": int(lpsim_plan_cut_lanes(g, p, k).sum()),
               "peak_loads": loads.tolist(), "peak_balance": round(float(loads.max() / loads.mean()), 4)}
        if args.steps:
            sim = Simulation(g, num_parts=k, node_part=p.ctypes.data, flags=0)
            sim.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
            sim.step(int(args.peak_s / 0.5))
            sim.step(args.steps)
            st = sim.stats()
            row.update(us_per_step=round(1e3 * st["step_ms"] / args.steps, 2), on_road=st["on_road"])
            sim.close()
        print(json.dumps(row), flush=True)
