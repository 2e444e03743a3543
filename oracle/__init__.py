"""Python handle on the plain-C CPU oracle (oracle/lpsim_oracle.c).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2406_08496_b200``) never imports it and
shares no code with it.

This module is argument marshalling only (ctypes); every step of the oracle's
arithmetic is in lpsim_oracle.c, which cites the paper passage it follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "liblpsim_oracle.so")
SO_OMP = os.path.join(HERE, "liblpsim_oracle_omp.so")
SRC = os.path.join(HERE, "lpsim_oracle.c")

CFLAGS = ["-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]


def build(force: bool = False, openmp: bool = False) -> str:
    """Compile the oracle (plain gcc; no FMA contraction).  openmp=True: the OpenMP variant used only
    for the CPU-baseline timing (same arithmetic; the per-trip loop runs on all host cores)."""
    so = SO_OMP if openmp else SO
    if force or not os.path.exists(so) or os.path.getmtime(so) < max(
        os.path.getmtime(SRC), os.path.getmtime(os.path.join(HERE, "lpsim_oracle.h"))
    ):
        tmp = so + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", *CFLAGS, *(["-fopenmp"] if openmp else []), "-o", tmp, SRC, "-lm"])
        os.replace(tmp, so)
    return so


class Params(C.Structure):
    _fields_ = [
        ("dt", C.c_float),
        ("a", C.c_float), ("b", C.c_float), ("s0", C.c_float), ("T", C.c_float),
        ("delta", C.c_int32),
        ("x0", C.c_float),
        ("g_a", C.c_float), ("g_b", C.c_float),
        ("alpha_i", C.c_float), ("alpha_a", C.c_float), ("alpha_b", C.c_float),
        ("sigma_a", C.c_float), ("sigma_b", C.c_float),
        ("h_min", C.c_int32), ("h_max", C.c_int32), ("lc_window", C.c_int32),
        ("signal_cycle_s", C.c_float), ("vfree", C.c_int32), ("reserved", C.c_int32),
        ("seed", C.c_uint64),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("step", C.c_int64), ("waiting", C.c_int64), ("on_road", C.c_int64),
        ("finished", C.c_int64), ("updates", C.c_int64), ("departures", C.c_int64),
        ("transitions", C.c_int64), ("lane_changes", C.c_int64), ("arrivals", C.c_int64),
        ("lost_claims", C.c_int64), ("digest", C.c_uint64),
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib = None
_lib_omp = None


def lib(openmp: bool = False):
    global _lib, _lib_omp
    if openmp:
        if _lib_omp is None:
            _lib_omp = _declare(C.CDLL(build(openmp=True)))
        return _lib_omp
    if _lib is None:
        _lib = _declare(C.CDLL(build()))
    return _lib


def _declare(l):
    if True:
        P = C.c_void_p
        l.lo_default_params.argtypes = [C.POINTER(Params)]
        l.lo_create.restype = P
        l.lo_create.argtypes = [C.c_int32, C.c_int32, P, P, P, P, P, P, C.POINTER(Params), C.c_char_p, C.c_int32]
        l.lo_load_demand.restype = C.c_int32
        l.lo_load_demand.argtypes = [P, C.c_int64, P, P, P, C.c_char_p, C.c_int32]
        l.lo_step.restype = C.c_int64
        l.lo_step.argtypes = [P, C.c_int64]
        l.lo_stats_get.argtypes = [P, C.POINTER(Stats)]
        l.lo_results.restype = C.c_int32
        l.lo_results.argtypes = [P, C.c_int64, P, P, P]
        l.lo_edge_entry.restype = C.c_int32
        l.lo_edge_entry.argtypes = [P, C.c_int64, P]
        l.lo_trip_state.restype = C.c_int32
        l.lo_trip_state.argtypes = [P, C.c_int64, P, P, P, P, P, P]
        l.lo_lane_map_size.restype = C.c_int64
        l.lo_lane_map_size.argtypes = [P]
        l.lo_lane_map_dump.restype = C.c_int32
        l.lo_lane_map_dump.argtypes = [P, P, C.c_int64]
        l.lo_h_max.restype = C.c_int32
        l.lo_h_max.argtypes = [P]
        l.lo_probe_trip.restype = C.c_int32
        l.lo_probe_trip.argtypes = [P, C.c_int64, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        l.lo_set_state.restype = C.c_int32
        l.lo_set_state.argtypes = [P, C.c_int64, C.c_int64, P, P, P, P, P, P, P]
        l.lo_destroy.argtypes = [P]
        l.lo_lane_map_layout.argtypes = [C.c_int32, P, P, P, C.POINTER(C.c_uint64)]
        l.lo_idm_accel.restype = C.c_float
        l.lo_idm_accel.argtypes = [C.POINTER(Params), C.c_float, C.c_float, C.c_int32, C.c_int32, C.c_int32]
        l.lo_philox4x32_10.argtypes = [P, P, P]
        l.lo_u24.restype = C.c_float
        l.lo_u24.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32]
        l.lo_eps.restype = C.c_float
        l.lo_eps.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_float]
        l.lo_depart_step.restype = C.c_int64
        l.lo_depart_step.argtypes = [C.c_double, C.c_float]
    return l


def default_params(**overrides) -> Params:
    p = Params()
    lib().lo_default_params(C.byref(p))
    for k, v in overrides.items():
        setattr(p, k, v)
    return p


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


class OracleError(RuntimeError):
    pass


class Oracle:
    """One oracle simulation: create -> load_demand -> step* -> results."""

    def __init__(self, graph, params: Params | None = None, openmp: bool = False):
        """openmp=True: the OpenMP build (CPU-baseline timing only; same results)."""
        self._l = lib(openmp)
        self._keep = []
        self.params = params or default_params()
        g = graph
        row_ptr = np.ascontiguousarray(g["row_ptr"], dtype=np.int64)
        dst = np.ascontiguousarray(g["dst"], dtype=np.int32)
        length = np.ascontiguousarray(g["length_m"], dtype=np.float32)
        lanes = np.ascontiguousarray(g["lanes"], dtype=np.uint8)
        v0 = np.ascontiguousarray(g["speed_limit_mps"], dtype=np.float32)
        self.n_edges = int(dst.shape[0])
        xy = g.get("node_xy")
        xy = np.ascontiguousarray(xy, dtype=np.float32).reshape(-1) if xy is not None and len(xy) else None
        self._keep.append(xy)
        err = C.create_string_buffer(512)
        h = self._l.lo_create(int(row_ptr.shape[0] - 1), self.n_edges, _ptr(row_ptr), _ptr(dst),
                            _ptr(length), _ptr(lanes), _ptr(v0), _ptr(xy), C.byref(self.params), err, 512)
        if not h:
            raise OracleError(err.value.decode())
        self.h = C.c_void_p(h)
        self.n_trips = 0

    def load_demand(self, depart_s, route_ptr, route_edges):
        d = np.ascontiguousarray(depart_s, dtype=np.float64)
        rp = np.ascontiguousarray(route_ptr, dtype=np.int64)
        re = np.ascontiguousarray(route_edges, dtype=np.int32)
        err = C.create_string_buffer(512)
        rc = self._l.lo_load_demand(self.h, int(d.shape[0]), _ptr(d), _ptr(rp), _ptr(re), err, 512)
        if rc != 0:
            raise OracleError(err.value.decode())
        self.n_trips = int(d.shape[0])
        self.r_total = int(rp[-1]) if rp.shape[0] else 0

    def step(self, n: int = 1):
        rc = self._l.lo_step(self.h, int(n))
        if rc != 0:
            raise OracleError("oracle invariant violated at step %d" % (-rc - 1))

    def stats(self) -> dict:
        s = Stats()
        self._l.lo_stats_get(self.h, C.byref(s))
        return s.as_dict()

    def results(self):
        n = self.n_trips
        a = np.empty(n, np.int64)
        t = np.empty(n, np.float64)
        d = np.empty(n, np.float64)
        self._l.lo_results(self.h, n, _ptr(a), _ptr(t), _ptr(d))
        return a, t, d

    def edge_entry_steps(self):
        """t_start per route entry (Alg. 1): snapshot step of entering route edge j, -1 if not."""
        out = np.empty(self.r_total, np.int64)
        if self._l.lo_edge_entry(self.h, self.r_total, _ptr(out)) != 0:
            raise OracleError("lo_edge_entry failed")
        return out

    def trip_state(self):
        n = self.n_trips
        out = dict(status=np.empty(n, np.int32), edge=np.empty(n, np.int32), lane=np.empty(n, np.int32),
                   pos=np.empty(n, np.float32), v=np.empty(n, np.float32), cursor=np.empty(n, np.int64))
        self._l.lo_trip_state(self.h, n, *(_ptr(out[k]) for k in ("status", "edge", "lane", "pos", "v", "cursor")))
        return out

    def set_state(self, step, status, edge, lane, pos, v, cursor, arrival_step=None):
        """Place the simulation at snapshot `step` with the given per-trip state (test scaffolding)."""
        n = self.n_trips
        a = [np.ascontiguousarray(status, np.int32), np.ascontiguousarray(edge, np.int32),
             np.ascontiguousarray(lane, np.int32), np.ascontiguousarray(pos, np.float32),
             np.ascontiguousarray(v, np.float32), np.ascontiguousarray(cursor, np.int64)]
        arr = np.ascontiguousarray(arrival_step, np.int64) if arrival_step is not None else None
        rc = self._l.lo_set_state(self.h, int(step), n, *(_ptr(x) for x in a), _ptr(arr))
        if rc != 0:
            raise OracleError("set_state: bad state (trip %d)" % (rc - 1))

    def lane_map(self):
        n = self._l.lo_lane_map_size(self.h)
        out = np.empty(n, np.uint8)
        self._l.lo_lane_map_dump(self.h, _ptr(out), n)
        return out

    def h_max(self) -> int:
        return self._l.lo_h_max(self.h)

    def probe(self, trip_id: int):
        g, vf, same = C.c_int32(), C.c_int32(), C.c_int32()
        r = self._l.lo_probe_trip(self.h, int(trip_id), C.byref(g), C.byref(vf), C.byref(same))
        if r < 0:
            raise OracleError("trip not on road")
        return (g.value, vf.value, bool(same.value)) if r == 1 else None

    def close(self):
        if getattr(self, "h", None):
            self._l.lo_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- pure helpers (pins) ---------------------------------------------------

def lane_map_layout(lanes, length_m):
    lanes = np.ascontiguousarray(lanes, dtype=np.uint8)
    length = np.ascontiguousarray(length_m, dtype=np.float32)
    base = np.empty(lanes.shape[0], np.uint64)
    total = C.c_uint64()
    lib().lo_lane_map_layout(int(lanes.shape[0]), _ptr(lanes), _ptr(length), _ptr(base), C.byref(total))
    return base, int(total.value)


def idm_accel(params: Params, v, v0, has_leader, s=0, vf=0) -> float:
    return lib().lo_idm_accel(C.byref(params), v, v0, int(has_leader), int(s), int(vf))


def philox4x32_10(ctr, key):
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    o = np.empty(4, np.uint32)
    lib().lo_philox4x32_10(_ptr(c), _ptr(k), _ptr(o))
    return o


def u24(seed, trip_id, k, stream) -> float:
    return lib().lo_u24(seed, trip_id, k, stream)


def eps(seed, trip_id, k, stream, sigma) -> float:
    return lib().lo_eps(seed, trip_id, k, stream, sigma)


def depart_step(depart_s: float, dt: float) -> int:
    return lib().lo_depart_step(depart_s, dt)


def run(graph, demand, steps: int, params: Params | None = None):
    """Convenience: simulate `steps` steps and return (oracle, results)."""
    o = Oracle(graph, params)
    o.load_demand(demand["depart_s"], demand["route_ptr"], demand["route_edges"])
    o.step(steps)
    return o, o.results()
