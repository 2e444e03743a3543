"""Test-side helpers: tiny hand-built networks and an independent Philox.

Nothing here is simulation arithmetic of the method; the Philox4x32-10 below
is an independent re-implementation (Salmon et al., SC'11) pinned by the
published Random123 known-answer vectors in test_oracle_pins.py.
"""
import numpy as np

M32 = 0xFFFFFFFF


def philox4x32_10(ctr, key):
    c = [int(x) & M32 for x in ctr]
    k0, k1 = int(key[0]) & M32, int(key[1]) & M32
    for r in range(10):
        if r:
            k0 = (k0 + 0x9E3779B9) & M32
            k1 = (k1 + 0xBB67AE85) & M32
        p0 = 0xD2511F53 * c[0]
        p1 = 0xCD9E8D57 * c[2]
        c = [((p1 >> 32) ^ c[1] ^ k0) & M32, p1 & M32, ((p0 >> 32) ^ c[3] ^ k1) & M32, p0 & M32]
    return c


def graph_from_edges(n_nodes, edges, xy=None):
    """edges: list of (src, dst, length_m, lanes, v0) in the desired id order;
    must already be grouped by src ascending (CSR order)."""
    src = np.array([e[0] for e in edges], np.int64)
    assert np.all(np.diff(src) >= 0), "edges must be listed in CSR order"
    row_ptr = np.zeros(n_nodes + 1, np.int64)
    np.cumsum(np.bincount(src, minlength=n_nodes), out=row_ptr[1:])
    g = {
        "row_ptr": row_ptr,
        "dst": np.array([e[1] for e in edges], np.int32),
        "length_m": np.array([e[2] for e in edges], np.float32),
        "lanes": np.array([e[3] for e in edges], np.uint8),
        "speed_limit_mps": np.array([e[4] for e in edges], np.float32),
    }
    if xy is not None:
        g["node_xy"] = np.asarray(xy, np.float32).reshape(-1)
    return g


def demand_from_routes(routes, depart_s):
    rp = np.zeros(len(routes) + 1, np.int64)
    rp[1:] = np.cumsum([len(r) for r in routes])
    re = np.array([e for r in routes for e in r], np.int32)
    return {"depart_s": np.asarray(depart_s, np.float64), "route_ptr": rp, "route_edges": re}


def merge_network(len_in=100.0, len_out=200.0, v0=13.9):
    """Nodes 0,1 -> 2 -> 3: in-edges e0 (0->2), e1 (1->2); out-edge e2 (2->3);
    plus return edges so the graph is strongly connected (e3: 3->0, e4: 3->1).
    All single-lane."""
    edges = [
        (0, 2, len_in, 1, v0),   # e0
        (1, 2, len_in, 1, v0),   # e1
        (2, 3, len_out, 1, v0),  # e2
        (3, 0, 50.0, 1, v0),     # e3
        (3, 1, 50.0, 1, v0),     # e4
    ]
    return graph_from_edges(4, edges)


def lc_network(v0=13.9, length=100.0):
    """A -> B on a 2-lane edge e0; B has two out-edges e1 (rank 0) and e2
    (rank 1), each to C; C -> A closes the loop.  Allowed lanes on e0 toward
    e1 are [0, 0] (rank 0 of K = 2, L = 2), toward e2 are [1, 1]."""
    edges = [
        (0, 1, length, 2, v0),  # e0  A->B
        (1, 2, 100.0, 1, v0),   # e1  B->C rank 0
        (1, 2, 120.0, 1, v0),   # e2  B->C rank 1
        (2, 0, 50.0, 1, v0),    # e3  C->A
    ]
    return graph_from_edges(3, edges)


def cross_network(arm=100.0, v0=13.9, lanes=1):
    """A signalised 4-way node (Q30): centre 0 with arms W=1 (-arm, 0), N=2 (0, arm), E=3 (arm, 0),
    S=4 (0, -arm), an edge each way per arm (the centre has in-degree 4).  Edge ids in CSR order:
    0: 0->1, 1: 0->2, 2: 0->3, 3: 0->4, 4: 1->0, 5: 2->0, 6: 3->0, 7: 4->0."""
    edges = [(0, 1, arm, lanes, v0), (0, 2, arm, lanes, v0), (0, 3, arm, lanes, v0), (0, 4, arm, lanes, v0),
             (1, 0, arm, lanes, v0), (2, 0, arm, lanes, v0), (3, 0, arm, lanes, v0), (4, 0, arm, lanes, v0)]
    xy = [(0.0, 0.0), (-arm, 0.0), (0.0, arm), (arm, 0.0), (0.0, -arm)]
    return graph_from_edges(5, edges, xy)
