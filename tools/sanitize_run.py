"""Workload for compute-sanitizer: C1b through the C ABI, checked against the oracle.

  compute-sanitizer --tool {memcheck,racecheck,synccheck} python tools/sanitize_run.py [steps]

Uses no torch (ctypes only), so every kernel the sanitizer sees is the library's.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    import oracle
    from paper_2406_08496_b200 import FLAG_DIGESTS, Simulation
    from workloads import make_workload

    g, d, _ = make_workload("grid4b")
    for parts in (1, 3):
        sim = Simulation(g, flags=FLAG_DIGESTS, num_parts=parts, sort_every=16)
        sim.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
        sim.step(steps)
        dig = sim.digests(steps)
        o = oracle.Oracle(g)
        o.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
        ref = []
        for _ in range(steps):
            o.step(1)
            ref.append(o.stats()["digest"])
        bad = np.nonzero(dig != np.array(ref, np.uint64))[0]
        print("parts=%d steps=%d digests %s" % (parts, steps, "identical" if not bad.size else "DIFFER at %d" % bad[0]))
        sim.close()


if __name__ == "__main__":
    main()
