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

# phantom bytes: occupied lane-map cells without a vehicle, and vehicles whose cell is free
occ_cells = np.nonzero(m != 255)[0]
veh_cells = np.sort(cellv)
print("occupied cells", len(occ_cells), "vehicles", len(on), "unique vehicle cells", len(np.unique(veh_cells)))
ph = np.setdiff1d(occ_cells, veh_cells)
print("phantom occupied cells:", len(ph))
miss = np.setdiff1d(veh_cells, occ_cells)
print("vehicles on free cells:", len(miss))
# stopped vehicles mid-edge: their leaders (same lane, nearest ahead)
mid = np.nonzero((v == 0) & ~atend)[0]
print("stopped mid-edge", len(mid))
order = np.lexsort((p, l, e))
import collections
lead_gap = collections.Counter()
for a_, b_ in zip(order[:-1], order[1:]):
    if e[a_] == e[b_] and l[a_] == l[b_] and v[a_] == 0 and not atend[a_]:
        lead_gap[int(np.floor(p[b_]) - np.floor(p[a_]))] += 1
print("gap to leader of stopped mid-edge vehicles:", sorted(lead_gap.items())[:12])
# heads of stopped queues: stopped mid-edge vehicles with no vehicle ahead in lane within 10 cells
heads = []
for a_, b_ in zip(order[:-1], list(order[1:]) + [-1]):
    pass

# queue heads: stopped mid-edge vehicles whose lane has no vehicle within 2 cells ahead
key = e.astype(np.int64) * 64 + l
idx_sorted = order
heads = []
for t_, a_ in enumerate(idx_sorted):
    if v[a_] != 0 or atend[a_]:
        continue
    b_ = idx_sorted[t_ + 1] if t_ + 1 < len(idx_sorted) else -1
    same = b_ >= 0 and key[b_] == key[a_]
    gap = int(np.floor(p[b_]) - np.floor(p[a_])) if same else 10**9
    if gap > 2:
        heads.append((a_, gap, b_ if same else -1))
print("queue heads (stopped, leader > 2 cells or none):", len(heads))
for a_, gap, b_ in heads[:12]:
    i = on[a_]
    c = int(np.floor(p[a_]))
    lane0 = base[e[a_]] + l[a_] * L[e[a_]]
    ahead = m[lane0 + c + 1: lane0 + min(c + 12, L[e[a_]])]
    print("  trip", i, "edge", e[a_], "lanes", ln[e[a_]], "lane", l[a_], "pos", p[a_], "Lc", L[e[a_]], "gap", gap,
          "leader v", v[b_] if b_ >= 0 else None, "cells ahead", ahead.tolist(), "next", nxt[a_])
