"""Cost of the periodic locality sort (a9) inside lpsim_step, at the C4 AM peak.

Runs to 8:00 h, then times single steps with and without a sort boundary
(lpsim_step's own CUDA-event time) and a 128-step call (one sort period).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2406_08496_b200 import Simulation
    from workloads import make_workload

    g, d, meta = make_workload(sys.argv[1] if len(sys.argv) > 1 else "bay9m", cache_dir="/tmp/lpsim_cache")
    sim = Simulation(g)
    sim.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
    sim.step(57600)  # 8:00 h, a multiple of the sort period
    out = {"on_road": sim.stats()["on_road"]}
    t = []
    for _ in range(3):
        sim.step(126)
        sim.step(1)
        a = sim.stats()["step_ms"]
        sim.step(1)  # crosses the sort boundary
        b = sim.stats()["step_ms"]
        t.append((a, b))
    out["plain_step_ms"] = [x for x, _ in t]
    out["sort_step_ms"] = [y for _, y in t]
    for _ in range(2):
        sim.step(128)
        out.setdefault("period_128_ms_per_step", []).append(sim.stats()["step_ms"] / 128)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
