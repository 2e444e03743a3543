"""The OpenMP build of the oracle (CPU baseline on all host cores) computes exactly what
the single-threaded parity build computes: same digest at every step, same results (-m "not gpu")."""
import numpy as np


def test_openmp_oracle_identical(oracle_mod):
    from workloads import make_workload

    g, d, _ = make_workload("grid4b", trips=1000, seed=3)
    out = []
    for omp in (False, True):
        o = oracle_mod.Oracle(g, openmp=omp)
        o.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
        dig = []
        for _ in range(900):
            o.step(1)
            dig.append(o.stats()["digest"])
        out.append((np.array(dig, np.uint64), o.results(), o.stats()))
    assert np.array_equal(out[0][0], out[1][0])
    for a, b in zip(out[0][1], out[1][1]):
        assert np.array_equal(a, b)
    assert out[0][2] == out[1][2]
