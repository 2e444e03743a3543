"""GPU parity on every path the step kernel can take, and the invariant checks.

* few CTAs (LPSIM_MAX_BLOCKS = 2 / 8 / 37): partitions with more than the two
  shared-memory-resident chunk rounds per CTA, so the HBM claim-record path
  (ClaimRec + the claimant ballot walk in phase C), the non-resident
  lane-change batch and the mid-loop flush of the lane-change queue run;
* fast roads (v0 = 40 m/s: H_max = 42 cells) and a 60-cell lane-change
  window: the multi-window scans (scan_first / scan_last) of the probe and of
  the gap acceptance;
* IDM exponent delta = 3 (the general exponentiation by squaring, Q6);
* the C4 AM-peak sample the bench's CPU baseline uses, digests every step;
* LPSIM_FLAG_CHECKS: a clean run, and a corrupted lane map reported as
  LPSIM_E_INVARIANT.

Every comparison is against the CPU oracle (oracle/), element by element.
"""
import os

import numpy as np
import pytest

from tests.conftest import cuda_available
from tests.test_gpu_parity import compare_results, run_pair

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]


class max_blocks:
    """LPSIM_MAX_BLOCKS is read by lpsim_create: CTAs of the step kernel."""

    def __init__(self, n):
        self.n = n

    def __enter__(self):
        self.old = os.environ.get("LPSIM_MAX_BLOCKS")
        os.environ["LPSIM_MAX_BLOCKS"] = str(self.n)

    def __exit__(self, *a):
        if self.old is None:
            os.environ.pop("LPSIM_MAX_BLOCKS", None)
        else:
            os.environ["LPSIM_MAX_BLOCKS"] = self.old


@pytest.mark.parametrize("ctas", [2, 8, 37])
def test_few_ctas_c1b(ctas):
    from workloads import make_workload

    g, d, _ = make_workload("grid4b")
    with max_blocks(ctas):
        sim, o = run_pair(g, d, 1500, check_every=300)
    compare_results(sim, o)


@pytest.mark.parametrize("ctas,flags", [(2, None), (8, None), (37, None), (2, 0)])
def test_few_ctas_sfcity(ctas, flags):
    """sfcity, 30k trips: with 2 CTAs a CTA holds ~20 chunk rounds of vehicles at the peak."""
    from workloads import make_workload

    g, d, _ = make_workload("sfcity", trips=30000)
    kw = {} if flags is None else dict(flags=flags)  # flags=0: the lean kernel (states only)
    with max_blocks(ctas):
        sim, o = run_pair(g, d, 2400, check_every=400, sim_kwargs=kw)
    compare_results(sim, o)


def test_few_ctas_partitions():
    """3 in-process partitions on 8 CTAs (each partition a few CTAs: multi-round paths + phase X)."""
    from workloads import make_workload

    g, d, _ = make_workload("sfcity", trips=20000)
    with max_blocks(8):
        sim, o = run_pair(g, d, 1500, check_every=500, sim_kwargs=dict(num_parts=3))
    compare_results(sim, o)


def _fast_grid(v0):
    from workloads import make_workload

    g, d, _ = make_workload("grid4b", trips=800, seed=5)
    g = dict(g)
    g["speed_limit_mps"] = np.full_like(g["speed_limit_mps"], v0)
    return g, d


def test_fast_roads_long_windows():
    """v0 = 40 m/s (probe windows up to 42 cells: more than one 48-byte window after alignment) and a
    60-cell lane-change window (121 cells: the scan_first / scan_last fallbacks)."""
    import oracle

    g, d = _fast_grid(40.0)
    sim, o = run_pair(g, d, 1200, check_every=200, sim_kwargs=dict(lc_window=60),
                      params=oracle.default_params(lc_window=60))
    compare_results(sim, o)
    s = o.stats()
    assert s["lane_changes"] > 0 and s["transitions"] > 0


def test_idm_delta_3():
    import oracle
    from workloads import make_workload

    g, d, _ = make_workload("grid4b", trips=600, seed=4)
    sim, o = run_pair(g, d, 1200, check_every=300, sim_kwargs=dict(delta=3), params=oracle.default_params(delta=3))
    compare_results(sim, o)


@pytest.mark.slow
def test_c4_peak_sample_digests():
    """The bench's CPU-baseline sample of C4 (trips departing in the 10 minutes after 8:00 h, shifted to
    t = 0; ~190k trips on the full Bay graph): digests every step for 1,800 steps, then the state."""
    import bench
    from workloads import make_workload

    g, d, _ = make_workload("bay9m", cache_dir=os.environ.get("LPSIM_CACHE", "/tmp/lpsim_cache"))
    s = bench.peak_sample(g, d, 8 * 3600.0, 600.0)
    sim, o = run_pair(g, s, 1800, check_every=900)
    compare_results(sim, o)
    assert o.stats()["on_road"] > 20000


def test_checks_flag_clean_run():
    from paper_2406_08496_b200 import FLAG_CHECKS, FLAG_DIGESTS
    from workloads import make_workload

    g, d, _ = make_workload("grid4b")
    sim, o = run_pair(g, d, 1200, check_every=400, sim_kwargs=dict(flags=FLAG_DIGESTS | FLAG_CHECKS))
    compare_results(sim, o)


def test_checks_flag_reports_corruption():
    """A stray byte in M_k (no vehicle owns it, so nothing clears it): the step after reports
    LPSIM_E_INVARIANT (the occupied cells no longer match the on-road vehicles), and the context
    refuses further steps."""
    from paper_2406_08496_b200 import FLAG_CHECKS, LpsimError, Simulation
    from workloads import make_workload

    g, d, _ = make_workload("grid4b")
    sim = Simulation(g, flags=FLAG_CHECKS)
    sim.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
    sim.step(300)
    m = sim.lane_map()
    free = np.nonzero(m == 255)[0]
    cell = int(free[len(free) // 2])
    sim.lpsim_debug_poke_map(cell, 7)
    with pytest.raises(LpsimError) as ei:
        sim.step(1)
    assert ei.value.status == 9, ei.value  # LPSIM_E_INVARIANT
    assert "step" in str(ei.value)
    with pytest.raises(LpsimError) as ei:
        sim.step(1)
    assert ei.value.status == 4  # LPSIM_E_STATE: unusable after the error


def test_checks_flag_catches_double_occupancy():
    """A stray byte a few cells ahead of a moving vehicle stays in its lane-map buffer (no vehicle owns
    it): when the buffer comes back as M_{k+2}, a vehicle writing its byte over it is caught by the
    per-step atomic check (naming the cell); if none reaches it, the count check after the call."""
    from paper_2406_08496_b200 import FLAG_CHECKS, LpsimError, Simulation
    from workloads import make_workload

    g, d, _ = make_workload("grid4b")
    sim = Simulation(g, flags=FLAG_CHECKS)
    sim.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
    sim.step(400)
    st = sim.trip_state()
    base = sim.lane_map_base()
    m = sim.lane_map()
    on = np.nonzero(st["status"] == 1)[0]
    order = on[np.argsort(-st["v"][on])]
    for i in order:  # the fastest vehicle with a free cell 4 ahead on its lane
        e, l, p = int(st["edge"][i]), int(st["lane"][i]), float(st["pos"][i])
        Lc = int(np.ceil(g["length_m"][e]))
        c = int(p) + 4
        if c < Lc and m[int(base[e]) + l * Lc + c] == 255:
            break
    sim.lpsim_debug_poke_map(int(base[e]) + l * Lc + c, 3)
    with pytest.raises(LpsimError) as ei:
        sim.step(3)
    assert ei.value.status == 9, ei.value  # LPSIM_E_INVARIANT
