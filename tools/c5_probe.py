"""Where does the C5 demand (24M trips) get stuck?  (diagnostic for DESIGN.md §5)

Runs the workload to 2x its horizon (or until drained) and classifies the vehicles still on the road:
edge class (speed limit / lanes), position (at the stop line or not), the downstream node's degrees,
and how the stuck vehicles cluster (connected components of the edges they occupy).
  python tools/c5_probe.py [--workload bay24m] [--trips N]
"""
import argparse
import collections
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="bay24m")
    ap.add_argument("--trips", type=int, default=None)
    ap.add_argument("--overrides", default="{}")
    args = ap.parse_args()
    from paper_2406_08496_b200 import Simulation
    from workloads import make_workload

    g, d, meta = make_workload(args.workload, trips=args.trips, cache_dir=os.environ.get("LPSIM_CACHE", "/tmp/lpsim_cache"),
                               **json.loads(args.overrides))
    sim = Simulation(g)
    sim.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
    horizon = int(meta["horizon_s"] / 0.5)
    hist = []
    steps = 0
    while steps < 2 * horizon:
        sim.step(7200)
        steps += 7200
        s = sim.stats()
        hist.append((steps // 7200, int(s["on_road"]), int(s["waiting"]), int(s["finished"])))
        if steps >= horizon and s["on_road"] == 0 and s["waiting"] == 0:
            break
    print(json.dumps({"workload": args.workload, "trips": meta["trips"], "hourly_on_road": hist}), flush=True)
    st = sim.trip_state()
    on = np.nonzero(st["status"] == 1)[0]
    if not len(on):
        print("drained")
        return
    e = st["edge"][on]
    L = np.ceil(g["length_m"]).astype(np.int64)
    sp = g["speed_limit_mps"]
    ln = g["lanes"].astype(int)
    src = np.repeat(np.arange(len(g["row_ptr"]) - 1), np.diff(g["row_ptr"]))
    dst = g["dst"]
    indeg = np.bincount(dst, minlength=len(g["row_ptr"]) - 1)
    outdeg = np.diff(g["row_ptr"])
    atend = np.floor(st["pos"][on]) >= L[e] - 1
    cls = collections.Counter((float(sp[x]), int(ln[x])) for x in e)
    print("stuck", len(on), "at stop line", int(atend.sum()), "v=0", int((st["v"][on] == 0).sum()))
    print("edge classes (speed, lanes):", cls.most_common(12))
    print("downstream (indeg, outdeg):", collections.Counter(zip(indeg[dst[e]].tolist(), outdeg[dst[e]].tolist())).most_common(10))
    # clusters of stuck edges (undirected components over the edges occupied by stuck vehicles)
    edges = np.unique(e)
    parent = {}

    def find(x):
        while parent.setdefault(x, x) != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x
    for x in edges:
        a, b = find(int(src[x])), find(int(dst[x]))
        if a != b:
            parent[a] = b
    comp = collections.Counter(find(int(src[x])) for x in e)
    sizes = sorted(comp.values(), reverse=True)
    print("clusters", len(sizes), "largest", sizes[:10])
    xy = g["node_xy"].reshape(-1, 2)
    for root, cnt in comp.most_common(5):
        nodes = [int(dst[x]) for x in edges if find(int(src[x])) == root]
        c = xy[nodes].mean(0)
        es = [x for x in edges if find(int(src[x])) == root]
        print("  cluster at (%.0f, %.0f) km: %d vehicles on %d edges, classes %s" % (
            c[0] / 1e3, c[1] / 1e3, cnt, len(es), collections.Counter((float(sp[x]), int(ln[x])) for x in es).most_common(4)))


if __name__ == "__main__":
    main()
