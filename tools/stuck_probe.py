"""Why are vehicles still on the road at the end of a run? (diagnostic)"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_08496_b200 import Simulation
from workloads import make_workload

g, d, meta = make_workload("bay", cache_dir="/tmp/lpsim_cache")
sim = Simulation(g)
sim.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
sim.step(24 * 7200)
st = sim.trip_state()
m = sim.lane_map()
L = np.ceil(g["length_m"]).astype(np.int64)
ln = g["lanes"].astype(np.int64)
base = np.concatenate([[0], np.cumsum(L * ln)])[:-1]
on = np.nonzero(st["status"] == 1)[0]
print("on road", len(on))
e = st["edge"][on]; l = st["lane"][on]; p = st["pos"][on]; v = st["v"][on]; cur = st["cursor"][on]
atend = np.floor(p) >= L[e] - 1
print("at stop line", atend.sum(), "speed 0", (v == 0).sum(), "at line & v0", (atend & (v == 0)).sum())
rp, re = d["route_ptr"], d["route_edges"]
nxt = np.array([re[rp[i] + c + 1] if rp[i] + c + 1 < rp[i + 1] else -1 for i, c in zip(on, cur)])
has = nxt >= 0
l2 = np.minimum(l, ln[np.maximum(nxt, 0)] - 1)
cell0 = base[np.maximum(nxt, 0)] + l2 * L[np.maximum(nxt, 0)]
occ0 = np.where(has, m[cell0] != 255, False)
print("at line, next entry occupied:", (atend & occ0).sum(), " free:", (atend & ~occ0 & has).sum())
# who occupies those entry cells? vehicles at cell 0 with speed?
oc = cell0[atend & occ0]
print("entry bytes (speed):", np.bincount(np.minimum(m[oc], 10)))
# chains: vehicle at line blocked by a vehicle at cell 0 that is itself blocked?
cellv = base[e] + l * L[e] + np.floor(p).astype(np.int64)
pos_of_cell = dict(zip(cellv.tolist(), range(len(on))))
blk = [pos_of_cell.get(int(c), -1) for c in oc]
blk = np.array(blk)
print("blockers found among on-road:", (blk >= 0).sum(), "of", len(blk))
if (blk >= 0).any():
    bb = blk[blk >= 0]
    print("blocker speeds", np.bincount(np.minimum(v[bb].astype(int), 10)), "blocker at its cell", np.bincount(np.minimum(np.floor(p[bb]).astype(int), 10)))
    # blocker's own situation: leader within its lane?
    print("sample blocker states:")
    for j in bb[:10]:
        i = on[j]
        print("  trip", i, "edge", e[j], "lane", l[j], "pos", p[j], "v", v[j], "Lc", L[e[j]], "cursor", cur[j], "routelen", rp[i+1]-rp[i])
