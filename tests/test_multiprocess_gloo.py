"""World-size-2 CPU (gloo) tests of the multi-process host logic (§8(e)).

Each rank derives the partition and the static exchange plan on its own from
the same inputs (SPMD); the tests check that the ranks agree, that the IPC
record exchange delivers every rank's record in rank order, and that the
per-rank results combine into the single-partition answer.
"""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # pragma: no cover - reported by the parent
        q.put((rank, "ERROR: %r" % (e,)))
    finally:
        dist.destroy_process_group()


def run_world(fn, world=2):
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for r, v in res.items():
        assert not (isinstance(v, str) and v.startswith("ERROR")), v
    return [res[r] for r in range(world)]


def plan_fn(rank, world):
    import torch
    import torch.distributed as dist

    from paper_2406_08496_b200 import build
    from paper_2406_08496_b200.lpsim import lpsim_partition_rcb, lpsim_plan_cut_lanes
    from paper_2406_08496_b200.multi import route_weights
    from workloads import make_workload

    build.build()
    g, d, _ = make_workload("sfcity", trips=20000)
    n = g["row_ptr"].shape[0] - 1
    part = lpsim_partition_rcb(n, g["node_xy"], route_weights(g, d), world)
    plan = lpsim_plan_cut_lanes(g, part, world)
    t = torch.from_numpy(part.astype(np.int64))
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t)
    same_part = all(bool((o == t).all()) for o in outs)
    pt = torch.from_numpy(plan.reshape(-1))
    outs = [torch.empty_like(pt) for _ in range(world)]
    dist.all_gather(outs, pt)
    same_plan = all(bool((o == pt).all()) for o in outs)
    # rank p's outgoing lanes to q are rank q's incoming from p (alltoall of the row / column views)
    send = [torch.tensor([int(plan[rank, q])]) for q in range(world)]
    recv = [torch.empty(1, dtype=torch.int64) for _ in range(world)]
    for q in range(world):  # gloo has no alltoall: emulate with send/recv pairs
        if q == rank:
            recv[q] = send[q]
            continue
        if rank < q:
            dist.send(send[q], q)
            dist.recv(recv[q], q)
        else:
            dist.recv(recv[q], q)
            dist.send(send[q], q)
    incoming_ok = all(int(recv[q]) == int(plan[q, rank]) for q in range(world))
    # the built-in multilevel partition is identical on every rank (deterministic per seed)
    from paper_2406_08496_b200.lpsim import lpsim_partition_multilevel
    ml = torch.from_numpy(lpsim_partition_multilevel(g, world, node_weight=route_weights(g, d), imbalance=0.05,
                                                     seed=1).astype(np.int64))
    outs = [torch.empty_like(ml) for _ in range(world)]
    dist.all_gather(outs, ml)
    same_part = same_part and all(bool((o == ml).all()) for o in outs)
    return dict(same_part=same_part, same_plan=same_plan, incoming_ok=incoming_ok,
                cut=int(plan.sum()), sizes=np.bincount(part, minlength=world).tolist())


def test_partition_and_plan_agree_across_ranks():
    res = run_world(plan_fn, 2)
    for r in res:
        assert r["same_part"] and r["same_plan"] and r["incoming_ok"]
        assert r["cut"] > 0
    assert res[0]["sizes"] == res[1]["sizes"] and min(res[0]["sizes"]) > 0


def blob_fn(rank, world):
    from paper_2406_08496_b200.multi import all_gather_blobs

    blob = bytes([rank]) * 7 + bytes(505)
    got = all_gather_blobs(blob)
    return [b[:8] for b in got]


def test_ipc_record_exchange_in_rank_order():
    res = run_world(blob_fn, 2)
    for r in res:
        assert r == [bytes([0]) * 7 + b"\0", bytes([1]) * 7 + b"\0"]


def combine_fn(rank, world):
    from paper_2406_08496_b200.multi import combine_results

    # trip i held by rank i % 2: arrival on the holder, -1 elsewhere; distance likewise
    n = 10
    a = np.where(np.arange(n) % world == rank, np.arange(n) * 10, -1)
    dd = np.where(np.arange(n) % world == rank, np.arange(n) * 1.5, 0.0)
    ca, cd = combine_results(a, dd)
    return ca.tolist(), cd.tolist()


def test_combine_results():
    res = run_world(combine_fn, 2)
    for ca, cd in res:
        assert ca == [i * 10 for i in range(10)]
        assert cd == [i * 1.5 for i in range(10)]
