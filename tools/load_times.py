"""Wall time of lpsim_create and lpsim_load_demand on a workload (stage times on stderr with
LPSIM_LOAD_TIMES=1)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2406_08496_b200 import Simulation  # noqa: E402
from workloads import make_workload  # noqa: E402

g, d, meta = make_workload(sys.argv[1] if len(sys.argv) > 1 else "bay9m", cache_dir="/tmp/lpsim_cache")
for rep in range(int(os.environ.get("REPS", "1"))):
    t0 = time.perf_counter()
    sim = Simulation(g)
    t1 = time.perf_counter()
    sim.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
    t2 = time.perf_counter()
    print("create %.3f s, load_demand %.3f s, device bytes %d, host cores %d" % (
        t1 - t0, t2 - t1, sim.stats()["device_bytes"], os.cpu_count()), flush=True)
    sim.close()
