"""Host-side partition logic (no GPU): the built-in route-weighted RCB."""
import numpy as np
import pytest


@pytest.fixture(scope="module")
def part_fn():
    from paper_2406_08496_b200 import build

    build.build()
    from paper_2406_08496_b200.lpsim import lpsim_partition_rcb

    return lpsim_partition_rcb


@pytest.mark.parametrize("k", [1, 2, 3, 4, 7, 8])
def test_rcb_balanced_and_complete(part_fn, k):
    from workloads.synth import sfcity_graph

    g, _ = sfcity_graph()
    n = g["row_ptr"].shape[0] - 1
    rng = np.random.default_rng(k)
    w = rng.integers(0, 50, n).astype(np.float64)
    p = part_fn(n, g["node_xy"], w, k)
    assert p.min() == 0 and p.max() == k - 1
    loads = np.bincount(p, weights=w, minlength=k)
    assert loads.max() <= 1.1 * w.sum() / k + w.max()
    # spatially compact: each part's bounding box is a rectangle slice
    assert len(np.unique(p)) == k


def test_rcb_deterministic_and_zero_weights(part_fn):
    xy = np.array([[0, 0], [1, 0], [2, 0], [3, 0], [10, 0], [11, 0]], np.float32)
    w = np.array([1, 1, 0, 0, 1, 1], np.float64)
    a = part_fn(6, xy, w, 2)
    b = part_fn(6, xy, w, 2)
    assert np.array_equal(a, b)
    # unvisited nodes 2, 3 follow their coordinates (nearest subgraph)
    assert a[0] == a[1] and a[4] == a[5] and a[0] != a[4]
    assert a[2] == a[0]


def test_rcb_without_coordinates(part_fn):
    p = part_fn(100, None, None, 4)
    assert np.array_equal(p, np.repeat(np.arange(4), 25))


# ---- balanced multilevel k-way (§8(f) item 1) ----
def _ml():
    from paper_2406_08496_b200.lpsim import lpsim_partition_multilevel, lpsim_plan_cut_lanes

    return lpsim_partition_multilevel, lpsim_plan_cut_lanes


def _cut_lanes(plan, g, part, k):
    m = plan(g, part, k)
    return int(m.sum())


@pytest.mark.parametrize("k", [2, 3, 4, 8])
def test_multilevel_balanced_complete_and_cuts_fewer_lanes_than_rcb(part_fn, k):
    """Every part non-empty, vertex weight within the imbalance bound (plus one vertex), and on
    the city graph the multilevel cut is no worse than route-weighted RCB's (the point of the
    scheme: P:L413-421 cuts by graph structure, RCB by coordinates only)."""
    from paper_2406_08496_b200.multi import route_weights
    from workloads import make_workload

    ml, plan = _ml()
    g, d, _ = make_workload("sfcity", trips=20000)
    n = g["row_ptr"].shape[0] - 1
    w = route_weights(g, d).astype(np.float64)
    p = ml(g, k, node_weight=w, imbalance=0.05, seed=3)
    assert p.shape == (n,) and p.min() == 0 and p.max() == k - 1 and len(np.unique(p)) == k
    eps = 1e-6 * w.sum() / n
    loads = np.bincount(p, weights=w + eps, minlength=k)
    assert loads.max() <= 1.05 * (w + eps).sum() / k + w.max() + 1e-9
    r = part_fn(n, g["node_xy"], w, k)
    assert _cut_lanes(plan, g, p, k) <= _cut_lanes(plan, g, r, k)


def test_multilevel_grid_bisection_is_near_optimal():
    """Unit-weight 16 x 16 grid (two-way lanes): the optimal bisection cuts one row of 16 links
    in both directions (32 lanes); the multilevel result must be balanced within 3 % and cut at
    most 1.5 x that."""
    from tests.helpers import graph_from_edges

    ml, plan = _ml()
    s = 16
    edges = []
    for y in range(s):
        for x in range(s):
            u = y * s + x
            if x + 1 < s:
                edges += [(u, u + 1, 100.0, 1, 13.9), (u + 1, u, 100.0, 1, 13.9)]
            if y + 1 < s:
                edges += [(u, u + s, 100.0, 1, 13.9), (u + s, u, 100.0, 1, 13.9)]
    g = graph_from_edges(s * s, sorted(edges))
    p = ml(g, 2, imbalance=0.03, seed=1)
    sizes = np.bincount(p, minlength=2)
    assert sizes.max() <= 1.03 * s * s / 2 + 1
    assert _cut_lanes(plan, g, p, 2) <= 48


def test_multilevel_deterministic_and_k1():
    from tests.helpers import graph_from_edges

    ml, _ = _ml()
    edges = [(i, i + 1, 50.0, 1, 13.9) for i in range(99)] + [(i + 1, i, 50.0, 2, 13.9) for i in range(99)]
    g = graph_from_edges(100, sorted(edges))
    a = ml(g, 4, seed=7)
    b = ml(g, 4, seed=7)
    assert np.array_equal(a, b)
    assert np.array_equal(ml(g, 1), np.zeros(100, np.int32))
    # a path splits into 4 contiguous runs: 3 cut links x 3 lanes (1 + 2 per direction)
    assert int(np.count_nonzero(np.diff(a))) == 3


def test_multilevel_rejects_bad_input():
    from paper_2406_08496_b200.lpsim import LpsimError
    from tests.helpers import graph_from_edges

    ml, _ = _ml()
    g = graph_from_edges(3, [(0, 1, 10.0, 1, 13.9), (1, 2, 10.0, 1, 13.9)])
    with pytest.raises(LpsimError):
        ml(g, 0)
    with pytest.raises(LpsimError):
        ml(g, 2, imbalance=-1.0)


# ---- unbalanced Leiden + k-means (§8(f) item 1) ----
def _two_cliques():
    """Two 6-cliques (two-way links, 1 lane) joined by one 2-lane two-way bridge 2 -> 8 / 8 -> 2;
    the cliques sit 1 km apart."""
    from tests.helpers import graph_from_edges

    edges = []
    for base in (0, 6):
        for a in range(6):
            for b in range(6):
                if a != b:
                    edges.append((base + a, base + b, 50.0, 1, 13.9))
    edges += [(2, 8, 500.0, 2, 13.9), (8, 2, 500.0, 2, 13.9)]
    xy = [(i % 3 * 10.0 + (1000.0 if i >= 6 else 0.0), i // 3 * 10.0) for i in range(12)]
    return graph_from_edges(12, sorted(edges), xy=xy)


def test_leiden_kmeans_separates_communities():
    from paper_2406_08496_b200.lpsim import lpsim_partition_leiden_kmeans, lpsim_plan_cut_lanes

    g = _two_cliques()
    p = lpsim_partition_leiden_kmeans(g, 2, seed=3)
    assert len(set(p[:6])) == 1 and len(set(p[6:])) == 1 and p[0] != p[6]
    assert int(lpsim_plan_cut_lanes(g, p, 2).sum()) == 4  # the bridge only, both directions
    assert np.array_equal(p, lpsim_partition_leiden_kmeans(g, 2, seed=3))
    # one part asked: everything together
    assert np.array_equal(lpsim_partition_leiden_kmeans(g, 1), np.zeros(12, np.int32))


@pytest.mark.parametrize("k", [2, 4])
def test_leiden_kmeans_city(k):
    """On the city graph: dense part ids, far fewer cut lanes than a random partition."""
    from paper_2406_08496_b200.lpsim import lpsim_partition_leiden_kmeans, lpsim_plan_cut_lanes
    from paper_2406_08496_b200.multi import route_weights
    from workloads import make_workload

    g, d, _ = make_workload("sfcity", trips=20000)
    n = g["row_ptr"].shape[0] - 1
    p = lpsim_partition_leiden_kmeans(g, k, node_weight=route_weights(g, d), seed=1)
    assert sorted(np.unique(p)) == list(range(k))
    r = np.random.default_rng(0).integers(0, k, n).astype(np.int32)
    assert lpsim_plan_cut_lanes(g, p, k).sum() * 10 < lpsim_plan_cut_lanes(g, r, k).sum()


def test_leiden_kmeans_needs_coordinates():
    from paper_2406_08496_b200.lpsim import LpsimError, lpsim_partition_leiden_kmeans

    g = _two_cliques()
    del g["node_xy"]
    with pytest.raises(LpsimError):
        lpsim_partition_leiden_kmeans(g, 2)


def test_occupancy_weights_count_vehicles_at_owner():
    """Pilot-run weights: one unit per on-road vehicle at the downstream node of its
    edge (the node whose partition owns the edge, §8(e)); waiting and finished trips count nothing."""
    from paper_2406_08496_b200.multi import occupancy_weights

    # 0 -> 1 (e0), 1 -> 2 (e1), 2 -> 0 (e2), 1 -> 0 (e3)
    g = {"row_ptr": np.array([0, 1, 3, 4]), "dst": np.array([1, 2, 0, 0])}
    status = np.array([1, 1, 1, 0, 2, 1])
    edge = np.array([0, 1, 3, 1, 1, 0])
    w = occupancy_weights(g, status, edge)
    assert w.tolist() == [1.0, 2.0, 1.0]
