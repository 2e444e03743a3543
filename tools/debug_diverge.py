"""Find the first step where GPU and oracle differ and print the differing trips."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_2406_08496_b200 import FLAG_DIGESTS, Simulation
from workloads import make_workload

name = sys.argv[1] if len(sys.argv) > 1 else "grid4b"
kw = {}
for a in sys.argv[2:]:
    k, v = a.split("=")
    kw[k] = int(v)
g, d, _ = make_workload(name)
sim = Simulation(g, flags=FLAG_DIGESTS, **kw)
sim.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
o = oracle.Oracle(g)
o.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
for k in range(3000):
    sim.step(1); o.step(1)
    gd = sim.digests(1)[0]; od = o.stats()["digest"]
    if gd != od:
        print("first divergence at snapshot", k + 1)
        gs, os_ = sim.trip_state(), o.trip_state()
        diff = np.nonzero((gs["status"] != os_["status"]) | ((os_["status"] == 1) & ((gs["edge"] != os_["edge"]) | (gs["lane"] != os_["lane"]) | (gs["pos"] != os_["pos"]) | (gs["v"] != os_["v"]) | (gs["cursor"] != os_["cursor"]))))[0]
        for i in diff[:20]:
            print(i, "gpu", {kk: gs[kk][i] for kk in gs}, "\n   ora", {kk: os_[kk][i] for kk in os_})
        print("stats gpu", sim.stats()); print("stats ora", o.stats())
        break
else:
    print("no divergence")
