"""Full-size C4 (BASELINE.json configs[3]: 9,008,766 trips, 147M cells) in the bench's launch
configuration (the lean step kernel, no instrumentation), checked by properties that hold at any
size — the oracle cannot run this workload, so the state is checked against the method's
invariants and closed forms, and partition invariance against a second, partitioned run:

* at the AM peak (8:00 h): the lane map M_k holds exactly one byte per on-road vehicle, at
  (edge, lane, floor(pos)) of its layout, equal to its speed floor(v);
  every other cell and the other lane-map buffer are free; conservation of trips;
* drained: every trip arrived, its distance is the sum of its route's edge lengths (exact in
  double, Q29 / DESIGN §1), it took at least one step per route edge after its departure step;
* the same demand on two partitions (one process, the exchange path) gives identical results.
"""
import os

import numpy as np
import pytest

from tests.conftest import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.slow,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def c4():
    from workloads import make_workload

    return make_workload("bay9m", cache_dir=os.environ.get("LPSIM_CACHE", "/tmp/lpsim_cache"))


def _drain(sim, trips, horizon_steps):
    steps = 0
    while True:
        sim.step(3600)
        steps += 3600
        if steps >= horizon_steps and sim.stats()["arrivals"] == trips:
            return steps
        assert steps < 3 * horizon_steps, "C4 did not drain"


def test_c4_full_size_properties(c4):
    from paper_2406_08496_b200 import Simulation

    g, d, meta = c4
    n = d["depart_s"].shape[0]
    sim = Simulation(g)  # lean kernel: the bench's
    sim.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
    k_peak = int(8 * 3600 / 0.5)
    sim.step(k_peak)
    st, ts = sim.stats(), sim.trip_state()
    on = np.nonzero(ts["status"] == 1)[0]
    assert st["on_road"] == on.size > 100_000
    assert st["waiting"] + st["on_road"] + st["finished"] == n
    assert st["finished"] == int((ts["status"] == 2).sum())
    # one byte per vehicle, at its cell, = floor(speed)
    m = sim.lane_map()
    base = sim.lane_map_base().astype(np.int64)
    Lc = np.ceil(np.asarray(g["length_m"], np.float32).astype(np.float64)).astype(np.int64)
    e, l = ts["edge"][on].astype(np.int64), ts["lane"][on].astype(np.int64)
    cell = base[e] + l * Lc[e] + np.floor(ts["pos"][on]).astype(np.int64)
    assert np.unique(cell).size == on.size, "two vehicles in one cell"
    assert np.array_equal(m[cell].astype(np.int64), np.minimum(np.floor(ts["v"][on]), 254).astype(np.int64))
    assert int((m != 255).sum()) == on.size
    occ = sim.lpsim_debug_map_occupancy()
    assert int(occ[0]) == on.size and int(occ[1]) == 0
    # drained: every trip arrived; distance = the route's length; >= one step per route edge
    _drain(sim, n, int(meta["horizon_s"] / 0.5))
    a, t, dist = sim.results()
    assert (a >= 0).all()
    rp = d["route_ptr"]
    lengths = np.asarray(g["length_m"], np.float32).astype(np.float64)  # the library's float lengths
    route_len = np.add.reduceat(lengths[d["route_edges"]], rp[:-1])
    assert np.array_equal(dist, route_len)
    dep_step = np.ceil(d["depart_s"] / 0.5 - 1e-9).astype(np.int64)  # smallest k with k*dt >= depart_s
    assert (a >= dep_step + np.diff(rp)).all()
    sim.close()


def test_c4_partition_invariance(c4):
    """Full C4 on one partition and on two (built-in multilevel partition, in-kernel exchange):
    identical arrival steps and distances for all 9.01M trips."""
    from paper_2406_08496_b200 import Simulation

    g, d, meta = c4
    n = d["depart_s"].shape[0]
    out = []
    for kw in (dict(), dict(num_parts=2)):
        sim = Simulation(g, **kw)
        sim.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
        _drain(sim, n, int(meta["horizon_s"] / 0.5))
        a, t, dist = sim.results()
        out.append((a, dist, sim.stats()["updates"]))
        sim.close()
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])
    assert out[0][2] == out[1][2]
