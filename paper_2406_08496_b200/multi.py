"""Multi-process plumbing for one-partition-per-GPU runs (§8(e)).

torch.distributed is used only to bootstrap (exchange the CUDA IPC records
of lpsim_ipc_handle) and to combine per-rank results; the per-step exchange
of migrants and entry halos happens inside the step kernel over NVLink peer
memory, with no host round trip.
"""
from __future__ import annotations

import numpy as np


def all_gather_blobs(blob: bytes, group=None) -> list[bytes]:
    """All-gather one fixed-size byte record per rank, in rank order (CPU / gloo)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    t = torch.frombuffer(bytearray(blob), dtype=torch.uint8)
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t, group=group)
    return [bytes(o.numpy().tobytes()) for o in outs]


def attach_peers(sim, group=None) -> None:
    """lpsim_ipc_handle on every rank, all-gather, lpsim_ipc_attach."""
    sim.ipc_attach(all_gather_blobs(sim.ipc_handle(), group))


def combine_results(arrival_step, distance_m, group=None):
    """Every trip is held by exactly one partition: element-wise max of the
    arrival steps (-1 elsewhere) and sum of the distances (0 elsewhere)."""
    import torch
    import torch.distributed as dist

    a = torch.from_numpy(np.ascontiguousarray(arrival_step, np.int64)).clone()
    d = torch.from_numpy(np.ascontiguousarray(distance_m, np.float64)).clone()
    dist.all_reduce(a, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(d, op=dist.ReduceOp.SUM, group=group)
    return a.numpy(), d.numpy()


def combine_edge_entry(edge_entry, group=None):
    """t_start per route entry: each entry is written by the one partition that resolved that
    departure or transition (-1 elsewhere): element-wise max."""
    import torch
    import torch.distributed as dist

    t = torch.from_numpy(np.ascontiguousarray(edge_entry, np.int32)).clone()
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t.numpy()


def combine_counts(stats: dict, keys=("updates", "departures", "transitions", "lane_changes", "arrivals",
                                      "lost_claims", "on_road", "finished"), group=None) -> dict:
    import torch
    import torch.distributed as dist

    v = torch.tensor([int(stats[k]) for k in keys], dtype=torch.int64)
    dist.all_reduce(v, op=dist.ReduceOp.SUM, group=group)
    out = dict(stats)
    out.update({k: int(x) for k, x in zip(keys, v.tolist())})
    return out


def route_weights(graph: dict, demand: dict) -> np.ndarray:
    """Route visit counts per node: the origin of every trip plus the
    downstream node of every route edge (host reference used by the tests)."""
    n = graph["row_ptr"].shape[0] - 1
    src = np.repeat(np.arange(n), np.diff(graph["row_ptr"]))
    w = np.zeros(n, np.float64)
    first = demand["route_edges"][demand["route_ptr"][:-1]]
    np.add.at(w, src[first], 1.0)
    np.add.at(w, graph["dst"][demand["route_edges"]], 1.0)
    return w


def occupancy_weights(graph: dict, status, edge) -> np.ndarray:
    """Vehicles on the road per node in one snapshot: each on-road vehicle counts for the downstream
    node of its edge, i.e. for the partition that owns the edge (§8(e) ownership).  The load the
    step kernel sees at that time, which route visits track only loosely at the peak: a
    congested edge holds many vehicles per visit."""
    n = graph["row_ptr"].shape[0] - 1
    on = np.asarray(status) == 1
    return np.bincount(np.asarray(graph["dst"])[np.asarray(edge)[on]], minlength=n).astype(np.float64)


def pilot_partition(graph: dict, demand: dict, k: int, t_s: float, device: int = 0, dt_s: float = 0.5,
                    imbalance: float = 0.03, seed: int = 1) -> np.ndarray:
    """A k-way multilevel partition (lpsim_partition_multilevel) balanced for the load at time t_s,
    measured by a one-partition pilot run of the same demand up to t_s (occupancy_weights).  The
    simulation is deterministic, so every rank that runs the pilot gets the same partition.
    Reading: the paper balances route visits; a traffic-assignment outer loop
     has the previous iteration's measured load, which balances the step itself."""
    from .lpsim import Simulation, lpsim_partition_multilevel

    sim = Simulation(graph, device=device, dt_s=dt_s)
    try:
        sim.load_demand(demand["depart_s"], demand["route_ptr"], demand["route_edges"])
        sim.step(int(round(t_s / dt_s)))
        ts = sim.trip_state()
    finally:
        sim.close()
    w = occupancy_weights(graph, ts["status"], ts["edge"])
    return lpsim_partition_multilevel(graph, k, node_weight=w, imbalance=imbalance, seed=seed)
