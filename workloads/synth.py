"""Seeded synthetic road graphs and routed OD demand (see package docstring).

Everything here is a pure function of (config, seed); numpy PCG64 draws.
No simulation arithmetic lives here.
"""
from __future__ import annotations

import ctypes as C
import hashlib
import os
import subprocess
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROUTE_SO = os.path.join(HERE, "libroute.so")
ROUTE_SRC = os.path.join(HERE, "route.c")


# --------------------------------------------------------------------------
# graph assembly helpers
# --------------------------------------------------------------------------

def _to_csr(n, src, dst, length, lanes, speed, key, xy):
    """Edges grouped by source node (CSR); within a node ordered by `key`."""
    src = np.asarray(src, np.int64)
    order = np.lexsort((np.arange(src.shape[0]), np.asarray(key, np.int64), src))
    src = src[order]
    row_ptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(src, minlength=n), out=row_ptr[1:])
    return {
        "row_ptr": row_ptr,
        "dst": np.asarray(dst, np.int32)[order],
        "length_m": np.asarray(length, np.float32)[order],
        "lanes": np.asarray(lanes, np.uint8)[order],
        "speed_limit_mps": np.asarray(speed, np.float32)[order],
        "node_xy": np.asarray(xy, np.float32).reshape(-1),
    }


def _largest_scc(n, src, dst):
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import connected_components

    m = csr_matrix((np.ones(len(src), np.int8), (src, dst)), shape=(n, n))
    _, lab = connected_components(m, directed=True, connection="strong")
    big = np.bincount(lab).argmax()
    keep = lab == big
    remap = -np.ones(n, np.int64)
    remap[keep] = np.arange(int(keep.sum()))
    return keep, remap


def graph_src(g):
    n = g["row_ptr"].shape[0] - 1
    return np.repeat(np.arange(n, dtype=np.int32), np.diff(g["row_ptr"]))


def graph_summary(g):
    return {
        "nodes": int(g["row_ptr"].shape[0] - 1),
        "edges": int(g["dst"].shape[0]),
        "cells": int((np.ceil(g["length_m"]).astype(np.int64) * g["lanes"]).sum()),
    }


# --------------------------------------------------------------------------
# C1: plain grid
# --------------------------------------------------------------------------

def grid_graph(nx=4, ny=4, spacing=100.0, lanes=2, speed=13.9):
    """nx·ny nodes, both directions between 4-neighbours; out-edges of a node
    in the order E, N, W, S.  2x2 -> 8 edges, 4x4 -> 48, 5x5 -> 80."""
    src, dst, key = [], [], []
    for y in range(ny):
        for x in range(nx):
            u = y * nx + x
            for d, (dx, dy) in enumerate(((1, 0), (0, 1), (-1, 0), (0, -1))):
                X, Y = x + dx, y + dy
                if 0 <= X < nx and 0 <= Y < ny:
                    src.append(u); dst.append(Y * nx + X); key.append(d)
    E = len(src)
    xy = np.array([(x * spacing, y * spacing) for y in range(ny) for x in range(nx)], np.float32)
    return _to_csr(nx * ny, src, dst, [spacing] * E, [lanes] * E, [speed] * E, key, xy)


# --------------------------------------------------------------------------
# C2 / C3: jittered city grids
# --------------------------------------------------------------------------

def _city_block(rng, nx, ny, gaps_x, gaps_y, origin, p_remove, p_oneway, art_every,
                local_speed, art_speed, lane_mix_local, lane_mix_art, fwy_every=0, fwy_skip=0,
                fwy_lanes=(3, 5), fwy_speed=29.0, jitter=0.1):
    """One jittered grid.  Returns node xy [n,2] and an edge table."""
    xs = origin[0] + np.concatenate([[0.0], np.cumsum(gaps_x)])
    ys = origin[1] + np.concatenate([[0.0], np.cumsum(gaps_y)])
    X, Y = np.meshgrid(xs, ys)  # [ny, nx]
    gx = np.concatenate([gaps_x[:1], gaps_x])
    gy = np.concatenate([gaps_y[:1], gaps_y])
    X = X + rng.uniform(-jitter, jitter, X.shape) * gx[None, :]
    Y = Y + rng.uniform(-jitter, jitter, Y.shape) * gy[:, None]
    xy = np.stack([X.ravel(), Y.ravel()], 1)
    nid = np.arange(nx * ny).reshape(ny, nx)

    segs = []  # (a, b, is_art, orient)
    # horizontal segments
    a = nid[:, :-1].ravel(); b = nid[:, 1:].ravel()
    row = np.repeat(np.arange(ny), nx - 1)
    segs.append((a, b, (row % art_every) == 0, np.zeros_like(a)))
    a = nid[:-1, :].ravel(); b = nid[1:, :].ravel()
    col = np.tile(np.arange(nx), ny - 1)
    segs.append((a, b, (col % art_every) == 0, np.ones_like(a)))
    A = np.concatenate([s[0] for s in segs]); B = np.concatenate([s[1] for s in segs])
    art = np.concatenate([s[2] for s in segs]); ori = np.concatenate([s[3] for s in segs])
    m = A.shape[0]
    keep = art | (rng.random(m) >= p_remove)
    oneway = (~art) & (rng.random(m) < p_oneway)
    flip = rng.random(m) < 0.5
    lanes_local = rng.choice(np.arange(1, len(lane_mix_local) + 1), size=m, p=lane_mix_local)
    lanes_art = rng.choice(np.arange(1, len(lane_mix_art) + 1), size=m, p=lane_mix_art)
    lanes = np.where(art, lanes_art, lanes_local)
    speed = np.where(art, art_speed, local_speed)
    A, B, lanes, speed, oneway, flip, ori = (t[keep] for t in (A, B, lanes, speed, oneway, flip, ori))
    # directions: both unless one-way
    s1, d1 = np.where(flip, B, A), np.where(flip, A, B)
    src = np.concatenate([s1, d1[~oneway]])
    dst = np.concatenate([d1, s1[~oneway]])
    ln = np.concatenate([lanes, lanes[~oneway]])
    sp = np.concatenate([speed, speed[~oneway]])
    # key: E, N, W, S by direction of travel
    dxy = xy[dst] - xy[src]
    horiz = np.concatenate([ori, ori[~oneway]]) == 0
    key = np.where(horiz, np.where(dxy[:, 0] > 0, 0, 2), np.where(dxy[:, 1] > 0, 1, 3))
    tables = [(src, dst, ln, sp, key)]
    extra_xy = []
    if fwy_every and fwy_skip:
        # Freeway corridors along every fwy_every-th row / column: two separate carriageways
        # (their own nodes, 60 m off the street) with an interchange every fwy_skip blocks:
        # an on-ramp from the street node and an off-ramp back to it.  A carriageway node
        # has two out-edges (continue = rank 0, off-ramp = rank 1), so through traffic
        # keeps half of the lanes at every interchange (Q14 splits lanes by out-edge rank).
        base_n = nx * ny
        fs, fd, fl, fsp, fk = [], [], [], [], []
        corridors = [("row", r) for r in range(fwy_every // 2, ny, fwy_every)] + \
                    [("col", c) for c in range(fwy_every // 2, nx, fwy_every)]
        for kind, rc in corridors:
            street = nid[rc, ::fwy_skip] if kind == "row" else nid[::fwy_skip, rc]
            if street.shape[0] < 2:
                continue
            lanes = int(rng.integers(fwy_lanes[0], fwy_lanes[1] + 1))
            for direction in (+1, -1):
                off = np.array([0.0, 60.0 * direction]) if kind == "row" else np.array([60.0 * direction, 0.0])
                fwy = []
                for g in street:
                    fwy.append(base_n + len(extra_xy))
                    extra_xy.append(xy[g] + off)
                order = list(range(len(street))) if direction > 0 else list(range(len(street)))[::-1]
                for a_, b_ in zip(order[:-1], order[1:]):  # carriageway links (rank 0 at their source)
                    fs.append(fwy[a_]); fd.append(fwy[b_]); fl.append(lanes); fsp.append(fwy_speed); fk.append(0)
                for q in range(len(street)):  # ramps
                    fs.append(street[q]); fd.append(fwy[q]); fl.append(2); fsp.append(15.6); fk.append(5)
                    fs.append(fwy[q]); fd.append(street[q]); fl.append(2); fsp.append(15.6); fk.append(1)
        if fs:
            tables.append((np.array(fs), np.array(fd), np.array(fl), np.array(fsp), np.array(fk)))
    if extra_xy:
        xy = np.concatenate([xy, np.array(extra_xy)])
    src = np.concatenate([t[0] for t in tables]); dst = np.concatenate([t[1] for t in tables])
    ln = np.concatenate([t[2] for t in tables]); sp = np.concatenate([t[3] for t in tables])
    key = np.concatenate([t[4] for t in tables])
    return xy, src, dst, ln, sp, key


def _finish_graph(xy, src, dst, ln, sp, key, min_len=5.0, max_len=3000.0):
    n = xy.shape[0]
    keep_n, remap = _largest_scc(n, src, dst)
    ok = keep_n[src] & keep_n[dst]
    src, dst, ln, sp, key = (t[ok] for t in (src, dst, ln, sp, key))
    L = np.linalg.norm(xy[dst] - xy[src], axis=1)
    L = np.clip(L, min_len, max_len)
    xy = xy[keep_n]
    g = _to_csr(xy.shape[0], remap[src], remap[dst], L, ln, sp, key, xy)
    return g, keep_n, remap


def sfcity_graph(seed=2, n=100):
    """C2: ~n x n jittered grid (110 m ±20 %), 15 % segments removed, 20 %
    one-way, arterials every 10th row/col (2-3 lanes, 15.6 m/s), locals 1-2
    lanes at 11.2 m/s; largest strongly connected component kept."""
    rng = np.random.default_rng(seed)
    gx = 110.0 * rng.uniform(0.8, 1.2, n - 1)
    gy = 110.0 * rng.uniform(0.8, 1.2, n - 1)
    xy, src, dst, ln, sp, key = _city_block(
        rng, n, n, gx, gy, (0.0, 0.0), p_remove=0.15, p_oneway=0.20, art_every=10,
        local_speed=11.2, art_speed=15.6, lane_mix_local=[0.7, 0.3], lane_mix_art=[0.0, 0.6, 0.4],
        jitter=0.05)
    g, keep_n, remap = _finish_graph(xy, src, dst, ln, sp, key)
    grid_ij = np.stack(np.meshgrid(np.arange(n), np.arange(n)), -1).reshape(-1, 2)[keep_n]
    return g, {"grid_ij": grid_ij, "block": [(0, n, n)]}


# county name, centre (km, x east / y north), population weight (millions)
BAY_COUNTIES = [
    ("sonoma", -32.0, 62.0, 0.49), ("napa", 2.0, 60.0, 0.14), ("solano", 32.0, 50.0, 0.45),
    ("marin", -22.0, 26.0, 0.26), ("contra_costa", 28.0, 24.0, 1.16), ("san_francisco", -12.0, 0.0, 0.87),
    ("alameda", 22.0, -6.0, 1.67), ("san_mateo", -6.0, -30.0, 0.77), ("santa_clara", 24.0, -52.0, 1.93),
]
# inter-county freeway corridors and bridges (bottlenecks)
BAY_LINKS = [
    ("san_francisco", "alameda", 5, "bay_bridge"), ("san_francisco", "marin", 3, "golden_gate"),
    ("san_mateo", "alameda", 3, "san_mateo_bridge"), ("marin", "contra_costa", 2, "richmond_bridge"),
    ("contra_costa", "solano", 4, "carquinez"), ("san_francisco", "san_mateo", 4, "us101"),
    ("san_mateo", "santa_clara", 4, "us101_south"), ("santa_clara", "alameda", 4, "i880"),
    ("alameda", "contra_costa", 4, "i680"), ("solano", "napa", 2, "sr12"),
    ("napa", "sonoma", 2, "sr12w"), ("sonoma", "marin", 3, "us101_north"),
]


def bay_graph(seed=3, target_nodes=224_223, fwy_every=48, fwy_skip=6, p_remove=0.38):
    """C3-C5: Bay-Area-shaped graph: nine county clusters of
    jittered grids sized by a population proxy; lognormal link lengths
    (median ~90 m); lane mix ~60/25/10/5 % of 1/2/3/4-5 lanes; freeway
    corridors (3-5 lanes, 29 m/s, multi-block links); bridges / corridors
    between counties as freeway chains of ~1 km links."""
    rng = np.random.default_rng(seed)
    tot_w = sum(c[3] for c in BAY_COUNTIES)
    inflate = 1.07  # the SCC prune drops a few % of grid nodes; freeway nodes come on top
    xys, tabs, blocks, grid_ij, county_of = [], [], [], [], []
    base = 0
    for ci, (name, cx, cy, w) in enumerate(BAY_COUNTIES):
        nn = int(target_nodes * inflate * w / tot_w)
        nx = max(8, int(np.sqrt(nn)))
        ny = max(8, nn // nx)
        mu, sig = np.log(90.0), 0.857
        gx = np.clip(rng.lognormal(mu, sig, nx - 1), 20.0, 600.0)
        gy = np.clip(rng.lognormal(mu, sig, ny - 1), 20.0, 600.0)
        origin = (cx * 1000.0 - gx.sum() / 2, cy * 1000.0 - gy.sum() / 2)
        xy, src, dst, ln, sp, key = _city_block(
            rng, nx, ny, gx, gy, origin, p_remove=p_remove, p_oneway=0.26, art_every=8,
            local_speed=11.2, art_speed=15.6, lane_mix_local=[0.68, 0.27, 0.05],
            lane_mix_art=[0.0, 0.45, 0.45, 0.10], fwy_every=fwy_every, fwy_skip=fwy_skip, jitter=0.1)
        xys.append(xy)
        tabs.append((src + base, dst + base, ln, sp, key))
        blocks.append((base, nx, ny))
        nfw = xy.shape[0] - nx * ny  # freeway carriageway nodes after the grid nodes
        grid_ij.append(np.concatenate([np.stack(np.meshgrid(np.arange(nx), np.arange(ny)), -1).reshape(-1, 2),
                                       np.full((nfw, 2), -1)]))
        county_of.append(np.full(xy.shape[0], ci))
        base += xy.shape[0]
    xy = np.concatenate(xys)
    names = [c[0] for c in BAY_COUNTIES]
    centre = {c[0]: np.array([c[1] * 1000.0, c[2] * 1000.0]) for c in BAY_COUNTIES}
    extra_xy, fs, fd, fl = [], [], [], []
    nxt = base
    for a, b, lanes, _ in BAY_LINKS:
        ia, ib = names.index(a), names.index(b)
        sa, sb = blocks[ia][0], blocks[ib][0]
        na, nb = blocks[ia][1] * blocks[ia][2], blocks[ib][1] * blocks[ib][2]
        pa = sa + np.argmin(np.linalg.norm(xy[sa:sa + na] - centre[b], axis=1))
        pb = sb + np.argmin(np.linalg.norm(xy[sb:sb + nb] - centre[a], axis=1))
        dist = np.linalg.norm(xy[pa] - xy[pb])
        k = max(1, int(dist // 1000.0))
        chain = [pa]
        for i in range(1, k):
            t = i / k
            extra_xy.append(xy[pa] * (1 - t) + xy[pb] * t)
            chain.append(nxt); nxt += 1
        chain.append(pb)
        for u, v in zip(chain[:-1], chain[1:]):
            fs += [u, v]; fd += [v, u]; fl += [lanes, lanes]
    if extra_xy:
        xy = np.concatenate([xy, np.array(extra_xy)])
    county_of.append(np.full(nxt - base, -1))
    src = np.concatenate([t[0] for t in tabs] + [np.array(fs)])
    dst = np.concatenate([t[1] for t in tabs] + [np.array(fd)])
    ln = np.concatenate([t[2] for t in tabs] + [np.array(fl)])
    sp = np.concatenate([t[3] for t in tabs] + [np.full(len(fs), 29.0)])
    key = np.concatenate([t[4] for t in tabs] + [np.full(len(fs), 5)])
    g, keep_n, remap = _finish_graph(xy, src.astype(np.int64), dst.astype(np.int64), ln, sp, key,
                                     max_len=3000.0)
    county = np.concatenate(county_of)[keep_n]
    gij = np.concatenate(grid_ij + [np.full((nxt - base, 2), -1)])[keep_n]
    return g, {"county": county, "grid_ij": gij, "names": names}


# --------------------------------------------------------------------------
# zones and demand
# --------------------------------------------------------------------------

def _zones_by_tiles(xy, n_zones, rng):
    """Zones = square tiles over the node cloud; the zone's centroid connector
    is the node nearest to the mean of its member nodes."""
    lo, hi = xy.min(0), xy.max(0)
    area = np.prod(hi - lo + 1.0)
    # tile size so that ~n_zones tiles are non-empty (nodes cover part of the box)
    side = np.sqrt(area / n_zones)
    for _ in range(30):
        ij = np.floor((xy - lo) / side).astype(np.int64)
        key = ij[:, 0] * 1_000_003 + ij[:, 1]
        uniq, zone = np.unique(key, return_inverse=True)
        if abs(len(uniq) - n_zones) <= 0.05 * n_zones:
            break
        side *= np.sqrt(len(uniq) / n_zones)
    nz = len(uniq)
    size = np.bincount(zone, minlength=nz).astype(np.float64)
    cen = np.stack([np.bincount(zone, xy[:, 0], nz), np.bincount(zone, xy[:, 1], nz)], 1) / size[:, None]
    conn = np.empty(nz, np.int64)
    order = np.argsort(zone, kind="stable")
    bounds = np.concatenate([[0], np.cumsum(np.bincount(zone, minlength=nz))])
    for z in range(nz):
        members = order[bounds[z]:bounds[z + 1]]
        conn[z] = members[np.argmin(np.linalg.norm(xy[members] - cen[z], axis=1))]
    return zone, size, cen, conn


def _gravity_od(rng, n_trips, size, cen, lam_m):
    """Origin zone ∝ size; destination ∝ size·exp(−dist/λ), d ≠ o."""
    nz = size.shape[0]
    o = rng.choice(nz, size=n_trips, p=size / size.sum())
    d = np.empty(n_trips, np.int64)
    order = np.argsort(o, kind="stable")
    counts = np.bincount(o, minlength=nz)
    starts = np.concatenate([[0], np.cumsum(counts)])
    for z in np.nonzero(counts)[0]:
        w = size * np.exp(-np.linalg.norm(cen - cen[z], axis=1) / lam_m)
        w[z] = 0.0
        cdf = np.cumsum(w)
        cdf /= cdf[-1]
        u = rng.random(counts[z])
        d[order[starts[z]:starts[z + 1]]] = np.minimum(np.searchsorted(cdf, u, side="right"), nz - 1)
    return o, d


def _peaked_departures(rng, n, horizon_s, peak_s, peak_sd_s, peak_share):
    t = rng.uniform(0.0, horizon_s, n)
    pk = rng.random(n) < peak_share
    m = int(pk.sum())
    x = rng.normal(peak_s, peak_sd_s, m)
    bad = (x < 0) | (x >= horizon_s)
    while bad.any():
        x[bad] = rng.normal(peak_s, peak_sd_s, int(bad.sum()))
        bad = (x < 0) | (x >= horizon_s)
    t[pk] = x
    return np.round(t, 1)  # decisecond resolution, like a trip table


# --------------------------------------------------------------------------
# routing (C helper)
# --------------------------------------------------------------------------

_route_lib = None


def _routelib():
    global _route_lib
    if _route_lib is None:
        if not os.path.exists(ROUTE_SO) or os.path.getmtime(ROUTE_SO) < os.path.getmtime(ROUTE_SRC):
            tmp = ROUTE_SO + ".tmp%d" % os.getpid()
            subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-pthread", "-o", tmp, ROUTE_SRC])
            os.replace(tmp, ROUTE_SO)
        l = C.CDLL(ROUTE_SO)
        P = C.c_void_p
        l.route_batch_begin.restype = P
        l.route_batch_begin.argtypes = [C.c_int32, C.c_int32, P, P, P, C.c_int64, P, P, P, P, P, C.c_int32]
        l.route_batch_finish.argtypes = [P, P, P]
        _route_lib = l
    return _route_lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def route_trips(g, origin, dest, threads=None):
    """Free-flow shortest paths (cost = round(1000·length/speed) ms); the parent
    of a node is its lowest-id tight in-edge.  Returns (route_ptr, route_edges)."""
    n = g["row_ptr"].shape[0] - 1
    E = g["dst"].shape[0]
    cost = np.maximum(1, np.round(1000.0 * g["length_m"].astype(np.float64)
                                  / g["speed_limit_mps"].astype(np.float64))).astype(np.int64)
    origin = np.asarray(origin, np.int32)
    dest = np.ascontiguousarray(dest, np.int32)
    trip_idx = np.argsort(origin, kind="stable").astype(np.int64)
    uo, counts = np.unique(origin[trip_idx], return_counts=True)
    group_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    group_origin = uo.astype(np.int32)
    route_len = np.empty(origin.shape[0], np.int64)
    row_ptr = np.ascontiguousarray(g["row_ptr"], np.int64)
    dst = np.ascontiguousarray(g["dst"], np.int32)
    threads = threads or max(1, min(64, os.cpu_count() or 1))
    h = _routelib().route_batch_begin(n, E, _p(row_ptr), _p(dst), _p(cost), len(uo), _p(group_origin),
                                      _p(group_ptr), _p(trip_idx), _p(dest), _p(route_len), threads)
    if (route_len <= 0).any():
        bad = int(np.nonzero(route_len <= 0)[0][0])
        _routelib().route_batch_finish(h, _p(np.zeros(origin.shape[0] + 1, np.int64)), None)
        raise ValueError("trip %d has no route" % bad)
    route_ptr = np.zeros(origin.shape[0] + 1, np.int64)
    np.cumsum(route_len, out=route_ptr[1:])
    route_edges = np.empty(int(route_ptr[-1]), np.int32)
    _routelib().route_batch_finish(h, _p(route_ptr), _p(route_edges))
    return route_ptr, route_edges


# --------------------------------------------------------------------------
# configs
# --------------------------------------------------------------------------

CONFIGS = {
    "grid4": dict(kind="grid", trips=1_000, horizon_s=3600.0, dep=(0.0, 3600.0), seed=1),
    "grid4b": dict(kind="grid", trips=1_000, horizon_s=3600.0, dep=(0.0, 300.0), seed=1),
    "sfcity": dict(kind="sfcity", trips=100_000, horizon_s=3 * 3600.0, zones=400, lam_m=2500.0, seed=2),
    # Bay: freeway corridors every 16 grid rows/cols; gravity decay 4.5 km (C3) / 3 km (C4) / 2.5 km
    # (C5), AM peak sd 1.75 / 2.5 / 4 h holding 50 / 50 / 20 % of the trips (chosen so that
    # every demand drains on this synthetic network: C5 with C4's 3 km / 50 % gridlocks the county
    # centres, 77 % of its trips arrive — tools/c5_probe.py)
    "bay": dict(kind="bay", trips=2_820_000, horizon_s=12 * 3600.0, zones=4000, lam_m=4500.0, seed=3,
                fwy_every=16, peak_sd_s=6300.0),
    "bay9m": dict(kind="bay", trips=9_008_766, horizon_s=12 * 3600.0, zones=4000, lam_m=3000.0, seed=4,
                  fwy_every=16, peak_sd_s=9000.0),
    "bay24m": dict(kind="bay", trips=24_000_000, horizon_s=24 * 3600.0, zones=4000, lam_m=2500.0, seed=5,
                   fwy_every=16, peak_sd_s=14400.0, peak_share=0.2),
}


def make_workload(name, trips=None, seed=None, threads=None, cache_dir=None, verbose=False, **overrides):
    """Returns (graph, demand, meta).  demand has depart_s, route_ptr,
    route_edges, origin, destination.  `trips` overrides the trip count (the
    graph stays the config's)."""
    cfg = dict(CONFIGS[name])
    if trips is not None:
        cfg["trips"] = int(trips)
    if seed is not None:
        cfg["seed"] = int(seed)
    cfg.update(overrides)
    key = hashlib.sha1(repr(sorted(cfg.items())).encode() + open(__file__, "rb").read()
                       + open(ROUTE_SRC, "rb").read()).hexdigest()[:16]
    if cache_dir:
        path = os.path.join(cache_dir, "%s_%s.npz" % (name, key))
        if os.path.exists(path):
            z = np.load(path)
            graph = {k[2:]: z[k] for k in z.files if k.startswith("g_")}
            demand = {k[2:]: z[k] for k in z.files if k.startswith("d_")}
            meta = dict(cfg, name=name, **graph_summary(graph), cached=True)
            return graph, demand, meta
    t0 = time.time()
    rng = np.random.default_rng(cfg["seed"])
    n_trips = cfg["trips"]
    if cfg["kind"] == "grid":
        graph = grid_graph(4, 4, 100.0, 2, 13.9)
        n = 16
        o = rng.integers(0, n, n_trips)
        d = (o + rng.integers(1, n, n_trips)) % n  # uniform over d != o
        dep = np.round(rng.uniform(cfg["dep"][0], cfg["dep"][1], n_trips), 1)
    else:
        if cfg["kind"] == "sfcity":
            graph, aux = sfcity_graph(seed=cfg["seed"])
            peak, sd, share = 1.5 * 3600.0, 0.5 * 3600.0, 0.5
        else:
            gkw = {k: cfg[k] for k in ("fwy_every", "fwy_skip", "p_remove") if k in cfg}
            graph, aux = bay_graph(seed=3, **gkw)  # one Bay graph for C3-C5
            peak, sd, share = 8.0 * 3600.0, cfg.get("peak_sd_s", 1.25 * 3600.0), cfg.get("peak_share", 0.5)
        xy = graph["node_xy"].reshape(-1, 2).astype(np.float64)
        zone, size, cen, conn = _zones_by_tiles(xy, cfg["zones"], rng)
        oz, dz = _gravity_od(rng, n_trips, size, cen, cfg["lam_m"])
        o, d = conn[oz], conn[dz]
        same = o == d  # two zones sharing a connector: move the destination
        while same.any():
            dz[same] = rng.integers(0, size.shape[0], int(same.sum()))
            d = conn[dz]
            same = o == d
        dep = _peaked_departures(rng, n_trips, cfg["horizon_s"], peak, sd, share)
    t1 = time.time()
    route_ptr, route_edges = route_trips(graph, o, d, threads=threads)
    t2 = time.time()
    demand = {
        "depart_s": dep.astype(np.float64),
        "route_ptr": route_ptr,
        "route_edges": route_edges,
        "origin": np.asarray(o, np.int32),
        "destination": np.asarray(d, np.int32),
    }
    meta = dict(cfg, name=name, **graph_summary(graph), gen_s=round(t1 - t0, 2), route_s=round(t2 - t1, 2),
                mean_route_edges=float(route_edges.shape[0] / max(1, n_trips)))
    if verbose:
        print(meta)
    if cache_dir:
        os.makedirs(cache_dir, exist_ok=True)
        tmp = path + ".tmp%d.npz" % os.getpid()
        np.savez(tmp, **{"g_" + k: v for k, v in graph.items()}, **{"d_" + k: v for k, v in demand.items()})
        os.replace(tmp, path)
    return graph, demand, meta
