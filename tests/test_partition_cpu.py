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
