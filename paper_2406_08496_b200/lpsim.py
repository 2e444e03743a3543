"""Thin ctypes binding of include/lpsim.h (argument marshalling only).

Every step of the simulated path runs in the sm_100a kernels of
``csrc/lpsim_step.cu`` behind the C ABI; this module converts numpy arrays to
pointers and status codes to exceptions.  It fails loudly when the CUDA
library is missing — there is no CPU fallback.

Names follow the C ABI: ``lpsim_create`` / ``lpsim_load_demand`` /
``lpsim_step`` / ``lpsim_results`` / ``lpsim_stats_get`` /
``lpsim_trip_state`` / ``lpsim_lane_map`` / ``lpsim_digests`` /
``lpsim_destroy``, wrapped by :class:`Simulation`.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LPSIM_LIB") or os.path.join(HERE, "liblpsim.so")

FLAG_DIGESTS = 0x1
FLAG_CHECKS = 0x2
FLAG_NO_SORT = 0x4
FLAG_TIMING = 0x8
FLAG_EDGE_TIMES = 0x10  # record t_start per route edge (set at creation)
FLAG_RACY = 0x20  # ablation: first-claimer-wins claims
FLAG_VFREE = 0x40  # ablation: literal v <- v_free

STATUS = {
    0: "LPSIM_OK", 1: "LPSIM_E_INVALID_ARG", 2: "LPSIM_E_INVALID_GRAPH", 3: "LPSIM_E_INVALID_DEMAND",
    4: "LPSIM_E_STATE", 5: "LPSIM_E_NOMEM", 6: "LPSIM_E_CAPACITY", 7: "LPSIM_E_CUDA", 8: "LPSIM_E_COMM",
    9: "LPSIM_E_INVARIANT",
}


class LpsimError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("%s: %s" % (STATUS.get(status, status), msg))
        self.status = status


class Graph(C.Structure):
    _fields_ = [
        ("struct_size", C.c_uint32), ("num_nodes", C.c_int32), ("num_edges", C.c_int32),
        ("row_ptr", C.c_void_p), ("dst", C.c_void_p), ("length_m", C.c_void_p), ("lanes", C.c_void_p),
        ("speed_limit_mps", C.c_void_p), ("node_xy", C.c_void_p),
    ]


class Config(C.Structure):
    _fields_ = [
        ("struct_size", C.c_uint32), ("dt_s", C.c_float),
        ("a", C.c_float), ("b", C.c_float), ("s0", C.c_float), ("T_headway", C.c_float),
        ("delta", C.c_int32), ("x0", C.c_float), ("g_a", C.c_float), ("g_b", C.c_float),
        ("alpha_i", C.c_float), ("alpha_a", C.c_float), ("alpha_b", C.c_float),
        ("sigma_a", C.c_float), ("sigma_b", C.c_float),
        ("h_min", C.c_int32), ("h_max", C.c_int32), ("lc_window", C.c_int32), ("sort_every", C.c_int32),
        ("seed", C.c_uint64), ("device", C.c_int32), ("num_parts", C.c_int32), ("node_part", C.c_void_p),
        ("stream", C.c_void_p), ("flags", C.c_uint32), ("rank", C.c_int32), ("world", C.c_int32),
        ("signal_cycle_s", C.c_float), ("reserved", C.c_int32 * 4),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("struct_size", C.c_uint32), ("step", C.c_int64), ("waiting", C.c_int64), ("on_road", C.c_int64),
        ("finished", C.c_int64), ("updates", C.c_int64), ("departures", C.c_int64), ("transitions", C.c_int64),
        ("lane_changes", C.c_int64), ("arrivals", C.c_int64), ("lost_claims", C.c_int64), ("digest", C.c_uint64),
        ("step_ms", C.c_double), ("exchange_ms", C.c_double), ("num_parts", C.c_int64),
        ("device_bytes", C.c_int64), ("kernel_launches", C.c_int64), ("phase_ns", C.c_int64 * 3),
        ("sort_ns", C.c_int64), ("soa_entries", C.c_int64),
    ]

    def as_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_ if f not in ("struct_size", "reserved", "phase_ns")}
        d["phase_ns"] = list(self.phase_ns)
        return d


_lib = None


def lib():
    """Load liblpsim.so (built by __graft_entry__.build()); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError("liblpsim.so not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        l = C.CDLL(LIB_PATH)
        P = C.c_void_p
        I = C.c_int
        l.lpsim_config_default.restype = I
        l.lpsim_config_default.argtypes = [C.POINTER(Config)]
        l.lpsim_create.restype = I
        l.lpsim_create.argtypes = [C.POINTER(Graph), C.POINTER(Config), C.POINTER(C.c_void_p)]
        l.lpsim_load_demand.restype = I
        l.lpsim_load_demand.argtypes = [P, C.c_int64, P, P, P, P, P]
        l.lpsim_step.restype = I
        l.lpsim_step.argtypes = [P, C.c_int64]
        l.lpsim_results.restype = I
        l.lpsim_results.argtypes = [P, C.c_int64, P, P, P]
        l.lpsim_stats_get.restype = I
        l.lpsim_stats_get.argtypes = [P, C.POINTER(Stats)]
        l.lpsim_trip_state.restype = I
        l.lpsim_trip_state.argtypes = [P, C.c_int64, P, P, P, P, P, P]
        l.lpsim_lane_map_size.restype = C.c_int64
        l.lpsim_lane_map_size.argtypes = [P]
        l.lpsim_lane_map.restype = I
        l.lpsim_lane_map.argtypes = [P, P, C.c_int64]
        l.lpsim_lane_map_base.restype = I
        l.lpsim_lane_map_base.argtypes = [P, P, C.c_int64]
        l.lpsim_digests.restype = I
        l.lpsim_digests.argtypes = [P, P, C.c_int64]
        l.lpsim_last_error.restype = C.c_char_p
        l.lpsim_last_error.argtypes = [P]
        l.lpsim_debug_block_times.restype = I
        l.lpsim_debug_block_times.argtypes = [P, P, C.c_int64]
        l.lpsim_debug_map_occupancy.restype = I
        l.lpsim_debug_map_occupancy.argtypes = [P, P]
        l.lpsim_debug_poke_map.restype = I
        l.lpsim_debug_poke_map.argtypes = [P, C.c_int64, C.c_uint8]
        l.lpsim_ipc_handle.restype = I
        l.lpsim_ipc_handle.argtypes = [P, P, C.c_int64]
        l.lpsim_ipc_attach.restype = I
        l.lpsim_ipc_attach.argtypes = [P, P, C.c_int64]
        l.lpsim_plan_cut_lanes.restype = I
        l.lpsim_plan_cut_lanes.argtypes = [C.POINTER(Graph), P, C.c_int32, P]
        l.lpsim_partition_rcb.restype = I
        l.lpsim_partition_rcb.argtypes = [C.c_int32, P, P, C.c_int32, P]
        l.lpsim_partition_leiden_kmeans.restype = I
        l.lpsim_partition_leiden_kmeans.argtypes = [C.POINTER(Graph), P, P, C.c_int32, C.c_double, C.c_uint64, P]
        l.lpsim_partition_multilevel.restype = I
        l.lpsim_partition_multilevel.argtypes = [C.POINTER(Graph), P, P, C.c_int32, C.c_double, C.c_uint64, P]
        l.lpsim_edge_entry_steps.restype = I
        l.lpsim_edge_entry_steps.argtypes = [P, C.c_int64, P]
        l.lpsim_restore.restype = I
        l.lpsim_restore.argtypes = [P, C.c_int64, C.c_int64, P, P, P, P, P, P, P, P, P]
        l.lpsim_set_flags.restype = I
        l.lpsim_set_flags.argtypes = [P, C.c_uint32]
        l.lpsim_destroy.restype = None
        l.lpsim_destroy.argtypes = [P]
        _lib = l
    return _lib


EXPORTED = [
    "lpsim_config_default", "lpsim_create", "lpsim_load_demand", "lpsim_step", "lpsim_results",
    "lpsim_stats_get", "lpsim_trip_state", "lpsim_lane_map_size", "lpsim_lane_map", "lpsim_lane_map_base",
    "lpsim_digests", "lpsim_partition_rcb", "lpsim_partition_multilevel", "lpsim_partition_leiden_kmeans", "lpsim_ipc_handle", "lpsim_ipc_attach", "lpsim_plan_cut_lanes",
    "lpsim_debug_block_times", "lpsim_debug_map_occupancy", "lpsim_debug_poke_map", "lpsim_set_flags", "lpsim_edge_entry_steps", "lpsim_restore", "lpsim_last_error", "lpsim_destroy",
]

IPC_BLOB_BYTES = 512


def _graph_struct(graph: dict):
    keep = {
        "row_ptr": np.ascontiguousarray(graph["row_ptr"], np.int64),
        "dst": np.ascontiguousarray(graph["dst"], np.int32),
        "length_m": np.ascontiguousarray(graph["length_m"], np.float32),
        "lanes": np.ascontiguousarray(graph["lanes"], np.uint8),
        "speed_limit_mps": np.ascontiguousarray(graph["speed_limit_mps"], np.float32),
    }
    xy = graph.get("node_xy")
    keep["node_xy"] = None if xy is None else np.ascontiguousarray(xy, np.float32)
    g = Graph(C.sizeof(Graph), int(keep["row_ptr"].shape[0] - 1), int(keep["dst"].shape[0]), _p(keep["row_ptr"]),
              _p(keep["dst"]), _p(keep["length_m"]), _p(keep["lanes"]), _p(keep["speed_limit_mps"]),
              _p(keep["node_xy"]))
    return g, keep


def lpsim_plan_cut_lanes(graph: dict, node_part, k: int):
    """Host-only: matrix [k, k] of cut lanes from upstream partition p to owner q."""
    g, keep = _graph_struct(graph)
    part = np.ascontiguousarray(node_part, np.int32)
    out = np.zeros(k * k, np.int64)
    rc = lib().lpsim_plan_cut_lanes(C.byref(g), _p(part), int(k), _p(out))
    if rc:
        raise LpsimError(rc, "lpsim_plan_cut_lanes")
    return out.reshape(k, k)


def lpsim_partition_rcb(num_nodes: int, node_xy=None, weight=None, k: int = 2):
    """Built-in route-weighted RCB partition (host-only, no device needed)."""
    xy = None if node_xy is None else np.ascontiguousarray(node_xy, np.float32)
    w = None if weight is None else np.ascontiguousarray(weight, np.float64)
    out = np.empty(num_nodes, np.int32)
    rc = lib().lpsim_partition_rcb(int(num_nodes), _p(xy), _p(w), int(k), _p(out))
    if rc:
        raise LpsimError(rc, "lpsim_partition_rcb")
    return out


def lpsim_partition_multilevel(graph: dict, k: int = 2, node_weight=None, edge_weight=None, imbalance: float = 0.03,
                               seed: int = 1):
    """Balanced multilevel k-way partition (host-only, no device needed); see include/lpsim.h."""
    g, keep = _graph_struct(graph)
    nw = None if node_weight is None else np.ascontiguousarray(node_weight, np.float64)
    ew = None if edge_weight is None else np.ascontiguousarray(edge_weight, np.float64)
    out = np.empty(int(g.num_nodes), np.int32)
    rc = lib().lpsim_partition_multilevel(C.byref(g), _p(nw), _p(ew), int(k), float(imbalance), int(seed), _p(out))
    if rc:
        raise LpsimError(rc, "lpsim_partition_multilevel")
    return out


def lpsim_partition_leiden_kmeans(graph: dict, k: int = 2, node_weight=None, edge_weight=None,
                                  resolution: float = 1.0, seed: int = 1):
    """Unbalanced Leiden communities + k-means partition (host-only); see include/lpsim.h."""
    g, keep = _graph_struct(graph)
    nw = None if node_weight is None else np.ascontiguousarray(node_weight, np.float64)
    ew = None if edge_weight is None else np.ascontiguousarray(edge_weight, np.float64)
    out = np.empty(int(g.num_nodes), np.int32)
    rc = lib().lpsim_partition_leiden_kmeans(C.byref(g), _p(nw), _p(ew), int(k), float(resolution), int(seed),
                                             _p(out))
    if rc:
        raise LpsimError(rc, "lpsim_partition_leiden_kmeans")
    return out


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def default_config(**overrides) -> Config:
    c = Config()
    c.struct_size = C.sizeof(Config)
    rc = lib().lpsim_config_default(C.byref(c))
    if rc:
        raise LpsimError(rc, "config_default")
    for k, v in overrides.items():
        setattr(c, k, v)
    return c


class Simulation:
    """One simulation context: lpsim_create -> lpsim_load_demand -> lpsim_step* ->
    lpsim_results / lpsim_stats_get -> lpsim_destroy."""

    def __init__(self, graph: dict, config: Config | None = None, **overrides):
        self.config = config or default_config()
        for k, v in overrides.items():
            setattr(self.config, k, v)
        g, self._keep = _graph_struct(graph)
        self.num_edges = int(self._keep["dst"].shape[0])
        h = C.c_void_p()
        rc = lib().lpsim_create(C.byref(g), C.byref(self.config), C.byref(h))
        if rc:
            raise LpsimError(rc, lib().lpsim_last_error(None).decode())
        self.h = h
        self.num_trips = 0

    def _check(self, rc):
        if rc:
            raise LpsimError(rc, lib().lpsim_last_error(self.h).decode())

    def lpsim_load_demand(self, depart_s, route_ptr, route_edges, origin=None, destination=None):
        d = np.ascontiguousarray(depart_s, np.float64)
        rp = np.ascontiguousarray(route_ptr, np.int64)
        re = np.ascontiguousarray(route_edges, np.int32)
        o = None if origin is None else np.ascontiguousarray(origin, np.int32)
        t = None if destination is None else np.ascontiguousarray(destination, np.int32)
        self._check(lib().lpsim_load_demand(self.h, int(d.shape[0]), _p(d), _p(rp), _p(re), _p(o), _p(t)))
        self.num_trips = int(d.shape[0])
        self.r_total = int(rp[-1]) if rp.shape[0] else 0

    load_demand = lpsim_load_demand

    def lpsim_step(self, n: int = 1):
        self._check(lib().lpsim_step(self.h, int(n)))

    step = lpsim_step

    def lpsim_results(self):
        n = self.num_trips
        a = np.empty(n, np.int64)
        t = np.empty(n, np.float64)
        d = np.empty(n, np.float64)
        self._check(lib().lpsim_results(self.h, n, _p(a), _p(t), _p(d)))
        return a, t, d

    results = lpsim_results

    def lpsim_stats_get(self) -> dict:
        s = Stats()
        s.struct_size = C.sizeof(Stats)
        self._check(lib().lpsim_stats_get(self.h, C.byref(s)))
        return s.as_dict()

    stats = lpsim_stats_get

    def lpsim_trip_state(self) -> dict:
        n = self.num_trips
        out = dict(status=np.empty(n, np.int32), edge=np.empty(n, np.int32), lane=np.empty(n, np.int32),
                   pos=np.empty(n, np.float32), v=np.empty(n, np.float32), cursor=np.empty(n, np.int64))
        self._check(lib().lpsim_trip_state(self.h, n, *(_p(out[k]) for k in
                                                         ("status", "edge", "lane", "pos", "v", "cursor"))))
        return out

    trip_state = lpsim_trip_state

    def lpsim_lane_map(self):
        n = lib().lpsim_lane_map_size(self.h)
        out = np.empty(n, np.uint8)
        self._check(lib().lpsim_lane_map(self.h, _p(out), n))
        return out

    lane_map = lpsim_lane_map

    def lpsim_lane_map_base(self):
        out = np.empty(self.num_edges, np.uint64)
        self._check(lib().lpsim_lane_map_base(self.h, _p(out), self.num_edges))
        return out

    lane_map_base = lpsim_lane_map_base

    def lpsim_digests(self, n: int):
        out = np.empty(n, np.uint64)
        self._check(lib().lpsim_digests(self.h, _p(out), int(n)))
        return out

    digests = lpsim_digests

    def lpsim_debug_block_times(self, grid_blocks: int):
        out = np.zeros(24 * grid_blocks, np.uint64)
        self._check(lib().lpsim_debug_block_times(self.h, _p(out), out.shape[0]))
        return out.reshape(grid_blocks, 24)

    def lpsim_debug_map_occupancy(self):
        """Occupied owned cells of (M_k, the other lane-map buffer); see include/lpsim.h."""
        out = np.zeros(2, np.uint64)
        self._check(lib().lpsim_debug_map_occupancy(self.h, _p(out)))
        return int(out[0]), int(out[1])

    def lpsim_debug_poke_map(self, cell: int, value: int):
        """Overwrite one byte of M_k (test instrumentation; see include/lpsim.h)."""
        self._check(lib().lpsim_debug_poke_map(self.h, int(cell), int(value)))

    def lpsim_edge_entry_steps(self):
        """t_start per route entry (Alg. 1): int32 [route_ptr[-1]], -1 = not entered."""
        out = np.empty(self.r_total, np.int32)
        self._check(lib().lpsim_edge_entry_steps(self.h, self.r_total, _p(out)))
        return out

    edge_entry_steps = lpsim_edge_entry_steps

    def checkpoint(self, edge_entry: bool = False) -> dict:
        """Snapshot of the whole simulation state at a step boundary: per-trip state,
        arrivals, counters (and t_start per route edge)."""
        st = self.trip_state()
        a, _, _ = self.results()
        s = self.stats()
        ck = dict(step=int(s["step"]), arrival_step=np.asarray(a, np.int64),
                  counters=np.array([s[k] for k in ("updates", "departures", "transitions", "lane_changes",
                                                    "arrivals", "lost_claims")], np.int64))
        ck.update({k: st[k] for k in ("status", "edge", "lane", "pos", "v", "cursor")})
        if edge_entry:
            ck["edge_entry"] = self.edge_entry_steps()
        return ck

    def lpsim_restore(self, ck: dict):
        a = {k: np.ascontiguousarray(ck[k], t) for k, t in (
            ("status", np.int32), ("edge", np.int32), ("lane", np.int32), ("pos", np.float32), ("v", np.float32),
            ("cursor", np.int64), ("arrival_step", np.int64), ("counters", np.int64))}
        ee = np.ascontiguousarray(ck["edge_entry"], np.int32) if ck.get("edge_entry") is not None else None
        self._check(lib().lpsim_restore(self.h, int(ck["step"]), int(a["status"].shape[0]), _p(a["status"]),
                                        _p(a["edge"]), _p(a["lane"]), _p(a["pos"]), _p(a["v"]), _p(a["cursor"]),
                                        _p(a["arrival_step"]), _p(a["counters"]), _p(ee)))

    restore = lpsim_restore

    def lpsim_set_flags(self, flags: int):
        self._check(lib().lpsim_set_flags(self.h, int(flags)))

    set_flags = lpsim_set_flags

    def lpsim_ipc_handle(self) -> bytes:
        buf = C.create_string_buffer(IPC_BLOB_BYTES)
        self._check(lib().lpsim_ipc_handle(self.h, C.cast(buf, C.c_void_p), IPC_BLOB_BYTES))
        return bytes(buf.raw)

    ipc_handle = lpsim_ipc_handle

    def lpsim_ipc_attach(self, blobs):
        data = b"".join(blobs)
        buf = C.create_string_buffer(data, len(data))
        self._check(lib().lpsim_ipc_attach(self.h, C.cast(buf, C.c_void_p), len(data)))

    ipc_attach = lpsim_ipc_attach

    def lpsim_destroy(self):
        if getattr(self, "h", None):
            lib().lpsim_destroy(self.h)
            self.h = None

    close = lpsim_destroy

    def __del__(self):
        try:
            self.lpsim_destroy()
        except Exception:
            pass
