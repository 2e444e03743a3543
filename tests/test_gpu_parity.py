"""GPU (C ABI) vs CPU oracle parity — the first gate.

Both sides run the same seeded inputs.  Integer state (status, edge, lane,
cell, cursor, departure / arrival step) is compared bit-exactly; fp32
positions and speeds are compared bit-exactly too (same fixed IEEE operation
order on both sides) although north_star only requires 1e-5 relative; the
per-snapshot order-independent digest is compared at every step so the first
divergent step is reported.
"""
import numpy as np
import pytest

from tests.conftest import cuda_available
from tests.helpers import demand_from_routes, graph_from_edges, lc_network, merge_network

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

REL_TOL = 1e-5  # north_star fp32 tolerance (relative, per step)


def run_pair(g, d, steps, check_every=0, sim_kwargs=None, params=None):
    import oracle
    from paper_2406_08496_b200 import FLAG_DIGESTS, Simulation

    kw = dict(flags=FLAG_DIGESTS)
    kw.update(sim_kwargs or {})
    sim = Simulation(g, **kw)
    sim.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
    o = oracle.Oracle(g, params)
    o.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
    done = 0
    chunk = check_every or steps
    digests = (kw["flags"] & FLAG_DIGESTS) != 0  # no digests: the lean step kernel (the bench's), states only
    while done < steps:
        n = min(chunk, steps - done)
        sim.step(n)
        if digests:
            gd = sim.digests(n)
            od = []
            for _ in range(n):
                o.step(1)
                od.append(o.stats()["digest"])
            od = np.array(od, np.uint64)
            bad = np.nonzero(gd != od)[0]
            assert bad.size == 0, "digest mismatch first at snapshot %d" % (done + bad[0] + 1)
        else:
            o.step(n)
        done += n
        if check_every:
            compare_state(sim, o)
    return sim, o


def compare_state(sim, o):
    gs, os_ = sim.trip_state(), o.trip_state()
    assert np.array_equal(gs["status"], os_["status"])
    on = os_["status"] == 1
    for k in ("edge", "lane", "cursor"):
        assert np.array_equal(gs[k][on], os_[k][on]), k
    for k in ("pos", "v"):
        a, b = gs[k][on].astype(np.float64), os_[k][on].astype(np.float64)
        assert np.all(np.abs(a - b) <= REL_TOL * np.maximum(1.0, np.abs(b))), k
        assert np.array_equal(gs[k][on], os_[k][on]), k + " (bit-exact)"
    assert np.array_equal(np.floor(gs["pos"][on]), np.floor(os_["pos"][on]))
    assert np.array_equal(sim.lane_map(), o.lane_map())


def compare_results(sim, o):
    a_g, t_g, d_g = sim.results()
    a_o, t_o, d_o = o.results()
    assert np.array_equal(a_g, a_o)
    assert np.array_equal(t_g, t_o)
    assert np.array_equal(d_g, d_o)
    s_g, s_o = sim.stats(), o.stats()
    for k in ("step", "waiting", "on_road", "finished", "updates", "departures", "transitions", "lane_changes",
              "arrivals", "lost_claims"):
        assert s_g[k] == s_o[k], (k, s_g[k], s_o[k])


def test_lane_map_layout_matches_oracle():
    import oracle
    from paper_2406_08496_b200 import Simulation
    from workloads import make_workload

    g, _, _ = make_workload("sfcity", trips=10)
    sim = Simulation(g)
    base_o, total_o = oracle.lane_map_layout(g["lanes"], g["length_m"])
    assert np.array_equal(sim.lane_map_base(), base_o)
    from paper_2406_08496_b200 import lib

    assert lib().lpsim_lane_map_size(sim.h) == total_o


@pytest.mark.parametrize("name", ["grid4", "grid4b"])
def test_c1_full_run(name):
    from workloads import make_workload

    g, d, _ = make_workload(name)
    sim, o = run_pair(g, d, 7200 + 1200, check_every=600)  # 1 h horizon + drain
    compare_results(sim, o)
    a, _, _ = sim.results()
    assert (a >= 0).all()


@pytest.mark.parametrize("name,steps,every", [("grid4b", 2400, 7), ("grid4", 7200 + 1200, 600)])
def test_lean_kernel(name, steps, every):
    """The lean step kernel (digest / timing code compiled out: the one bench.py times) against the
    oracle: full trip state and lane map at checkpoints, final results and counters."""
    from workloads import make_workload

    g, d, _ = make_workload(name)
    sim, o = run_pair(g, d, steps, check_every=every, sim_kwargs=dict(flags=0))
    compare_results(sim, o)


def test_set_flags_between_steps():
    """Switching between the lean and the instrumented step kernel mid-run (lpsim_set_flags, as the
    bench's exchange window does) leaves the results unchanged."""
    import oracle
    from paper_2406_08496_b200 import FLAG_TIMING, Simulation
    from workloads import make_workload

    g, d, _ = make_workload("grid4b")
    sim = Simulation(g, flags=0)
    sim.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
    o = oracle.Oracle(g)
    o.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
    for flags, n in ((0, 200), (FLAG_TIMING, 150), (0, 250)):
        sim.set_flags(flags)
        sim.step(n)
        o.step(n)
        compare_state(sim, o)
    st = sim.stats()
    assert st["exchange_ms"] == 0.0  # one partition


@pytest.mark.parametrize("name,trips,steps,kw", [
    ("grid4b", None, 2400, dict(flags=0)),
    ("grid4b", None, 2400, dict(num_parts=3)),
    ("sfcity", 20_000, 1500, dict(flags=0)),
])
def test_edge_entry_steps_match_oracle(name, trips, steps, kw):
    """t_start per route edge (Alg. 1, LPSIM_FLAG_EDGE_TIMES) is bit-exact against the
    oracle: lean kernel, partitions, city window."""
    from paper_2406_08496_b200 import FLAG_EDGE_TIMES
    from workloads import make_workload

    g, d, _ = make_workload(name, trips=trips)
    kw = dict(kw)
    kw["flags"] = kw.get("flags", 1) | FLAG_EDGE_TIMES
    sim, o = run_pair(g, d, steps, check_every=steps // 3, sim_kwargs=kw)
    ge, oe = sim.edge_entry_steps(), o.edge_entry_steps()
    assert ge.shape == oe.shape and (oe >= 0).sum() > 0
    assert np.array_equal(ge.astype(np.int64), oe)


@pytest.mark.parametrize("name,trips,steps,kw", [
    ("grid4b", None, 3000, dict()),
    ("grid4", None, 7200 + 1200, dict(flags=0)),
    ("grid4b", None, 2000, dict(num_parts=4)),
    ("sfcity", 20_000, 1500, dict()),
])
def test_signals_match_oracle(name, trips, steps, kw):
    """Signalised intersections (§8(f), Q30: fixed-cycle two-phase signals, 60 s) against the
    oracle: digests every step (instrumented kernel) or states at checkpoints (lean kernel), final
    results, counters and t_start per route edge."""
    import oracle
    from paper_2406_08496_b200 import FLAG_EDGE_TIMES
    from workloads import make_workload

    g, d, _ = make_workload(name, trips=trips)
    kw = dict(kw)
    kw["flags"] = kw.get("flags", 1) | FLAG_EDGE_TIMES
    kw["signal_cycle_s"] = 60.0
    sim, o = run_pair(g, d, steps, check_every=steps // 4, sim_kwargs=kw,
                      params=oracle.default_params(signal_cycle_s=60.0))
    compare_results(sim, o)
    assert np.array_equal(sim.edge_entry_steps().astype(np.int64), o.edge_entry_steps())


def test_edge_entry_needs_flag_at_create():
    from paper_2406_08496_b200 import FLAG_EDGE_TIMES, LpsimError, Simulation
    from workloads import make_workload

    g, d, _ = make_workload("grid4b", trips=10)
    sim = Simulation(g)
    sim.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
    with pytest.raises(LpsimError):
        sim.edge_entry_steps()
    with pytest.raises(LpsimError):
        sim.set_flags(FLAG_EDGE_TIMES)


def test_lean_kernel_sfcity_window():
    from workloads import make_workload

    g, d, _ = make_workload("sfcity", trips=20_000)
    sim, o = run_pair(g, d, 1500, check_every=250, sim_kwargs=dict(flags=0))
    compare_results(sim, o)


def test_c1b_state_every_step_early():
    from workloads import make_workload

    g, d, _ = make_workload("grid4b")
    sim, o = run_pair(g, d, 300, check_every=1)
    compare_results(sim, o)


@pytest.mark.parametrize("sort_every,flags_extra", [(1, 0), (3, 0), (16, 0), (0, 4)])
def test_order_independence(sort_every, flags_extra):
    """Results must not depend on SoA order: sort every step / rarely / never."""
    from paper_2406_08496_b200 import FLAG_DIGESTS
    from workloads import make_workload

    g, d, _ = make_workload("grid4b", trips=600, seed=7)
    sim, o = run_pair(g, d, 900, check_every=300,
                      sim_kwargs=dict(sort_every=sort_every, flags=FLAG_DIGESTS | flags_extra))
    compare_results(sim, o)


def test_shuffled_ids_not_sorted_by_departure():
    """Trip ids in random order w.r.t. departure: the pending-set minimum (A7)
    must still pick the lowest eligible id."""
    from workloads import make_workload

    g, d, _ = make_workload("grid4b", trips=800, seed=3)
    rng = np.random.default_rng(5)
    perm = rng.permutation(800)
    rl = np.diff(d["route_ptr"])
    routes = [d["route_edges"][d["route_ptr"][i]:d["route_ptr"][i + 1]] for i in perm]
    dd = demand_from_routes(routes, d["depart_s"][perm] * 0.2)  # dense: long departure queues
    sim, o = run_pair(g, dd, 1200, check_every=200)
    compare_results(sim, o)
    del rl


def test_deep_departure_queue():
    """Thousands of trips on one departure slot (3-level bitmap) with random ids."""
    g = merge_network(len_out=60.0)
    rng = np.random.default_rng(1)
    n = 2500
    routes = [[2] if rng.random() < 0.9 else [0, 2] for _ in range(n)]
    dep = rng.uniform(0, 400, n).round(1)
    d = demand_from_routes(routes, dep)
    sim, o = run_pair(g, d, 3000, check_every=500)
    compare_results(sim, o)


def test_merge_and_lane_change_scripts():
    g = merge_network()
    routes = [[3, 0]] * 3 + [[0, 2], [3, 0], [1, 2]]
    d = demand_from_routes(routes, [5000.0] * 3 + [0.0, 5000.0, 0.0])
    sim, o = run_pair(g, d, 100, check_every=1)
    compare_results(sim, o)
    assert o.stats()["lost_claims"] >= 1
    g = lc_network(length=300.0)
    rng = np.random.default_rng(2)
    routes = [[0, 1] if rng.random() < 0.5 else [0, 2] for _ in range(300)]
    d = demand_from_routes(routes, np.sort(rng.uniform(0, 200, 300)).round(1))
    sim, o = run_pair(g, d, 800, check_every=50)
    compare_results(sim, o)
    assert o.stats()["lane_changes"] > 10


def test_zero_trips_and_single_trip():
    g = graph_from_edges(2, [(0, 1, 100.0, 1, 13.9), (1, 0, 100.0, 1, 13.9)])
    d = demand_from_routes([], [])
    d["route_ptr"] = np.zeros(1, np.int64)
    sim, o = run_pair(g, d, 10)
    assert sim.stats()["updates"] == 0
    d = demand_from_routes([[0]], [0.0])
    sim, o = run_pair(g, d, 40, check_every=1)
    compare_results(sim, o)
    assert sim.results()[0][0] == 26  # SURVEY §8(c) worked case


def test_sfcity_window():
    from workloads import make_workload

    g, d, _ = make_workload("sfcity", trips=30000)
    sim, o = run_pair(g, d, 2400, check_every=400)
    compare_results(sim, o)


@pytest.mark.slow
def test_bay_fullsize_window():
    """Full-size Bay graph and demand (C3, the bench workload): parity over the
    first 1,200 steps (digest every step, full state at checkpoints)."""
    from workloads import make_workload

    g, d, _ = make_workload("bay", cache_dir="/tmp/lpsim_cache")
    sim, o = run_pair(g, d, 1200, check_every=400)
    compare_results(sim, o)


def test_invalid_inputs_fail_loudly():
    from paper_2406_08496_b200 import LpsimError, Simulation

    g = graph_from_edges(2, [(0, 1, 0.5, 1, 13.9), (1, 0, 100.0, 1, 13.9)])
    with pytest.raises(LpsimError) as ei:
        Simulation(g)
    assert ei.value.status == 2 and "index 0" in str(ei.value)
    g = graph_from_edges(2, [(0, 1, 10.0, 1, 13.9), (1, 0, 100.0, 1, 13.9)])
    sim = Simulation(g)
    with pytest.raises(LpsimError) as ei:
        sim.load_demand([0.0], [0, 2], [0, 0])  # 0 -> 1 then 0 again: not connected
    assert ei.value.status == 3
    with pytest.raises(LpsimError) as ei:
        sim.step(1)
    assert ei.value.status == 4


def test_invalid_demand_reports_first_offending_trip():
    """Demand validation runs on all host cores; the error still names the first offending trip."""
    from paper_2406_08496_b200 import LpsimError, Simulation

    g = graph_from_edges(2, [(0, 1, 10.0, 1, 13.9), (1, 0, 100.0, 1, 13.9)])
    n = 300_000
    dep = np.zeros(n)
    rp = np.arange(n + 1, dtype=np.int64) * 2
    re = np.tile(np.array([0, 1], np.int32), n)
    for bad in (0, 150_001, n - 1):
        re2 = re.copy()
        re2[2 * bad + 1] = 0  # 0 -> 1 then 0 again: not connected
        re2[2 * (n - 1) + 1] = 0 if bad == n - 1 else 1
        if bad < n - 1:
            re2[2 * 250_000 + 1] = 0  # a later bad trip must not be the one reported
        sim = Simulation(g)
        with pytest.raises(LpsimError) as ei:
            sim.load_demand(dep, rp, re2)
        assert ei.value.status == 3 and ("trip %d)" % bad) in str(ei.value), str(ei.value)


# ---------------------------------------------------------------------------
# partitions (§8(e)): identical results at any partition count
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("parts", [2, 3, 4, 8])
def test_partitions_match_oracle_grid(parts):
    from workloads import make_workload

    g, d, _ = make_workload("grid4b", trips=1000, seed=11)
    sim, o = run_pair(g, d, 1500, check_every=250, sim_kwargs=dict(num_parts=parts))
    compare_results(sim, o)
    assert sim.stats()["num_parts"] == parts


@pytest.mark.parametrize("parts", [2, 4, 8])
def test_partitions_match_oracle_sfcity(parts):
    from workloads import make_workload

    g, d, _ = make_workload("sfcity", trips=30000)
    sim, o = run_pair(g, d, 2400, check_every=800, sim_kwargs=dict(num_parts=parts))
    compare_results(sim, o)


def test_user_partition_and_random_partition():
    """Any node partition (even a random one) gives the same results."""
    from paper_2406_08496_b200 import FLAG_DIGESTS
    from workloads import make_workload

    g, d, _ = make_workload("grid4b", trips=800, seed=2)
    rng = np.random.default_rng(0)
    part = rng.integers(0, 5, 16).astype(np.int32)
    part[:5] = np.arange(5)
    sim, o = run_pair(g, d, 1200, check_every=300,
                      sim_kwargs=dict(num_parts=5, flags=FLAG_DIGESTS, node_part=part.ctypes.data))
    compare_results(sim, o)


@pytest.mark.parametrize("k,kind", [(2, "multilevel"), (4, "multilevel"), (4, "leiden")])
def test_multilevel_partition_matches_oracle(k, kind):
    """The balanced multilevel partition (§8(f) item 1, lpsim_partition_multilevel) and
    the unbalanced Leiden + k-means one, route-visit node weights, passed as
    node_part: results identical to the oracle."""
    from paper_2406_08496_b200 import FLAG_DIGESTS
    from paper_2406_08496_b200.lpsim import lpsim_partition_leiden_kmeans, lpsim_partition_multilevel
    from paper_2406_08496_b200.multi import route_weights
    from workloads import make_workload

    g, d, _ = make_workload("sfcity", trips=20000)
    fn = lpsim_partition_multilevel if kind == "multilevel" else lpsim_partition_leiden_kmeans
    part = fn(g, k, node_weight=route_weights(g, d), seed=5)
    assert len(np.unique(part)) == k
    sim, o = run_pair(g, d, 1500, check_every=500,
                      sim_kwargs=dict(num_parts=k, flags=FLAG_DIGESTS, node_part=part.ctypes.data))
    compare_results(sim, o)
    assert sim.stats()["num_parts"] == k


def test_pilot_partition_matches_oracle():
    """The partition balanced for the load at a given time (multi.pilot_partition: a one-partition
    pilot run to t, vehicles on the road per owning node as weights): deterministic, every
    part non-empty, and the K-partition run from t = 0 is identical to the oracle."""
    from paper_2406_08496_b200 import FLAG_DIGESTS
    from paper_2406_08496_b200.multi import pilot_partition
    from workloads import make_workload

    g, d, _ = make_workload("sfcity", trips=20000)
    part = pilot_partition(g, d, 4, 400.0)
    assert np.array_equal(part, pilot_partition(g, d, 4, 400.0))
    assert len(np.unique(part)) == 4
    sim, o = run_pair(g, d, 1500, check_every=500,
                      sim_kwargs=dict(num_parts=4, flags=FLAG_DIGESTS, node_part=part.ctypes.data))
    compare_results(sim, o)


# ---------------------------------------------------------------------------
# checkpoint / restore (§8(f) item 3): per-trip state is the whole state at a step boundary
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name,trips,k_ck,k_end,kw_a,kw_b", [
    ("grid4b", None, 700, 2400, dict(), dict()),
    ("grid4b", None, 333, 2000, dict(), dict(num_parts=3)),           # restored into 3 partitions
    ("grid4b", None, 900, 2400, dict(signal_cycle_s=60.0), dict(signal_cycle_s=60.0, flags=0)),
    ("sfcity", 20_000, 600, 1500, dict(), dict()),
])
def test_restore_matches_uninterrupted(name, trips, k_ck, k_end, kw_a, kw_b):
    import oracle
    from paper_2406_08496_b200 import FLAG_DIGESTS, FLAG_EDGE_TIMES, Simulation
    from workloads import make_workload

    g, d, _ = make_workload(name, trips=trips)
    args = (d["depart_s"], d["route_ptr"], d["route_edges"])
    a = Simulation(g, **dict(dict(flags=FLAG_EDGE_TIMES), **kw_a))
    a.load_demand(*args)
    a.step(k_ck)
    ck = a.checkpoint(edge_entry=True)
    a.step(k_end - k_ck)
    kb = dict(kw_b)
    kb["flags"] = kb.get("flags", FLAG_DIGESTS) | FLAG_EDGE_TIMES
    b = Simulation(g, **kb)
    b.load_demand(*args)
    b.restore(ck)
    sb = b.stats()
    assert sb["step"] == k_ck and sb["on_road"] == int((ck["status"] == 1).sum())
    b.step(k_end - k_ck)
    compare_state(b, _OracleView(a))
    for k in ("step", "waiting", "on_road", "finished", "updates", "departures", "transitions", "lane_changes",
              "arrivals", "lost_claims"):
        assert b.stats()[k] == a.stats()[k], k
    for x, y in zip(a.results(), b.results()):
        assert np.array_equal(x, y)
    assert np.array_equal(a.edge_entry_steps(), b.edge_entry_steps())
    # and the oracle's uninterrupted run
    o = oracle.Oracle(g, oracle.default_params(signal_cycle_s=kw_a.get("signal_cycle_s", 0.0)))
    o.load_demand(*args)
    o.step(k_end)
    compare_results(b, o)
    assert np.array_equal(b.edge_entry_steps().astype(np.int64), o.edge_entry_steps())


class _OracleView:
    """Adapter: a Simulation seen through the oracle's trip_state / lane_map interface."""

    def __init__(self, sim):
        self.sim = sim

    def trip_state(self):
        return self.sim.trip_state()

    def lane_map(self):
        return self.sim.lane_map()


def test_restore_state_checks():
    from paper_2406_08496_b200 import LpsimError, Simulation
    from workloads import make_workload

    g, d, _ = make_workload("grid4b", trips=200)
    args = (d["depart_s"], d["route_ptr"], d["route_edges"])
    a = Simulation(g)
    a.load_demand(*args)
    a.step(400)
    ck = a.checkpoint()
    with pytest.raises(LpsimError) as ei:  # not a fresh context
        a.restore(ck)
    assert ei.value.status == 4
    on = np.nonzero(ck["status"] == 1)[0]
    assert on.size > 0
    bad = dict(ck)
    bad["lane"] = ck["lane"].copy()
    bad["lane"][on[0]] = 7
    b = Simulation(g)
    b.load_demand(*args)
    with pytest.raises(LpsimError) as ei:
        b.restore(bad)
    assert ei.value.status == 1 and ("trip %d)" % on[0]) in str(ei.value)


# ---------------------------------------------------------------------------
# Ablations (§8(f) item 4)
# ---------------------------------------------------------------------------
def test_vfree_matches_oracle():
    """The literal "v <- v_free" (LPSIM_FLAG_VFREE) is deterministic: digests every step vs the oracle."""
    import oracle
    from paper_2406_08496_b200 import FLAG_DIGESTS, FLAG_VFREE
    from workloads import make_workload

    g, d, _ = make_workload("grid4b")
    sim, o = run_pair(g, d, 2400, check_every=600, sim_kwargs=dict(flags=FLAG_DIGESTS | FLAG_VFREE),
                      params=oracle.default_params(vfree=1))
    compare_results(sim, o)


def test_racy_claims_keep_invariants():
    """Paper-faithful racy claims (LPSIM_FLAG_RACY: first contender wins) are not reproducible,
    so they are checked by invariants: one vehicle per cell (the lane map's occupied bytes = on-road
    count), conservation, every trip drains, and the mean travel time stays within 5 % of the
    deterministic lowest-id rule's on the conflict-heavy C1b demand."""
    from paper_2406_08496_b200 import FLAG_RACY, Simulation
    from workloads import make_workload

    g, d, _ = make_workload("grid4b")
    res = {}
    for flags in (0, FLAG_RACY):
        sim = Simulation(g, flags=flags)
        sim.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
        for _ in range(12):
            sim.step(200)
            st = sim.stats()
            assert int((sim.lane_map() != 255).sum()) == st["on_road"]
            assert st["waiting"] + st["on_road"] + st["finished"] == 1000
        a, t, _ = sim.results()
        assert (a >= 0).all()
        res[flags] = float((t - d["depart_s"]).mean())
    assert abs(res[FLAG_RACY] - res[0]) <= 0.05 * res[0], res


@pytest.mark.parametrize("parts,sort_every", [(1, 128), (1, 1), (3, 16)])
def test_lane_map_buffers_clean_after_resolve(parts, sort_every):
    """a7: at every step boundary M_k holds exactly one cell per
    on-road vehicle, and the other buffer — M_k's cells cleared in the resolve phase, M_{k+2}
    next — is all free (checked over the owned edges of every partition; lean kernel, with
    arrivals, migrations between partitions and sorts dropping dead entries in between)."""
    from paper_2406_08496_b200 import Simulation
    from workloads import make_workload

    g, d, _ = make_workload("sfcity", trips=20_000)
    sim = Simulation(g, flags=0, num_parts=parts, sort_every=sort_every)
    sim.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
    seen_arrivals = False
    for n in (1, 2, 97, 400, 700, 1301):
        sim.step(n)
        occ, other = sim.lpsim_debug_map_occupancy()
        st = sim.stats()
        assert occ == st["on_road"], (st["step"], occ, st["on_road"])
        assert other == 0, (st["step"], other)
        seen_arrivals |= st["arrivals"] > 0
    assert seen_arrivals and st["on_road"] > 0
