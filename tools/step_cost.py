"""Per-step cost diagnostics: fixed cost (empty network), sort period effect."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2406_08496_b200 import FLAG_NO_SORT, FLAG_TIMING, Simulation
    from workloads import make_workload

    g, d, meta = make_workload("bay", cache_dir="/tmp/lpsim_cache")
    # fixed cost: no trips
    sim = Simulation(g)
    sim.load_demand(np.zeros(0), np.zeros(1, np.int64), np.zeros(0, np.int32))
    for n in (1, 16, 256, 4096):
        sim.step(n)
        s = sim.stats()
        print(json.dumps(dict(case="empty", steps_per_call=n, us_per_step=1e3 * s["step_ms"] / n)), flush=True)
    sim.close()
    for label, kw in (("sort128+timing", dict(flags=FLAG_TIMING)), ("sort16", dict(sort_every=16)),
                      ("nosort", dict(flags=FLAG_NO_SORT))):
        sim = Simulation(g, **kw)
        sim.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
        t0 = time.time()
        sim.step(7200)
        s = sim.stats()
        r = dict(case=label, t="0-1h", on_road=s["on_road"], us_per_step=1e3 * s["step_ms"] / 7200)
        sim.step(50400)  # to 8:00
        s = sim.stats()
        r["ffwd_us_per_step"] = 1e3 * s["step_ms"] / 50400
        sim.step(1024)
        s = sim.stats()
        r.update(peak_on_road=s["on_road"], peak_us_per_step=1e3 * s["step_ms"] / 1024, wall=time.time() - t0,
                 phase_us_per_step=[x / 1e3 / 1024 for x in s["phase_ns"]])
        for n in (1, 16):
            tt = 0.0
            for _ in range(8):
                sim.step(n)
                tt += sim.stats()["step_ms"]
            r["peak_us_per_step_calls_of_%d" % n] = 1e3 * tt / (8 * n)
        print(json.dumps(r), flush=True)
        sim.close()


if __name__ == "__main__":
    main()
