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
