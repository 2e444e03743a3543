"""Multi-process mode (one partition per process, CUDA IPC peer memory, flag
barriers in the step kernel) — two processes on ONE device (time-sliced), so
the real cross-process exchange path runs on a single-GPU box.  Results must
equal the oracle's."""
import os
import socket

import numpy as np
import pytest

from tests.conftest import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

STEPS = 400


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["LPSIM_MAX_BLOCKS"] = "148"
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2406_08496_b200 import FLAG_DIGESTS, FLAG_EDGE_TIMES, Simulation
        from paper_2406_08496_b200.multi import attach_peers, combine_edge_entry, combine_results
        from workloads import make_workload

        g, d, _ = make_workload("grid4b", trips=600, seed=9)
        sim = Simulation(g, device=0, rank=rank, world=world, flags=FLAG_DIGESTS | FLAG_EDGE_TIMES)
        sim.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
        attach_peers(sim)
        dist.barrier()
        sim.step(STEPS)
        dig = sim.digests(STEPS)
        a, t, dist_m = sim.results()
        ca, cd = combine_results(a, dist_m)
        ce = combine_edge_entry(sim.edge_entry_steps())
        q.put((rank, dict(dig=dig.tolist(), arrival=ca.tolist(), dist=cd.tolist(), entry=ce.tolist(),
                          stats=sim.stats())))
    except Exception as e:
        q.put((rank, "ERROR: %r" % (e,)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_processes_match_oracle(world):
    import multiprocessing as mp

    import oracle
    from workloads import make_workload

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
    g, d, _ = make_workload("grid4b", trips=600, seed=9)
    o = oracle.Oracle(g)
    o.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
    od = []
    for _ in range(STEPS):
        o.step(1)
        od.append(o.stats()["digest"])
    gd = [sum(int(res[r]["dig"][i]) for r in range(world)) % (1 << 64) for i in range(STEPS)]
    bad = [i for i in range(STEPS) if gd[i] != od[i]]
    assert not bad, "digest mismatch first at snapshot %d" % (bad[0] + 1)
    a_o, _, d_o = o.results()
    assert np.array_equal(np.array(res[0]["arrival"]), a_o)
    assert np.array_equal(np.array(res[0]["dist"]), d_o)
    assert np.array_equal(np.array(res[0]["entry"]), o.edge_entry_steps())  # t_start per route edge
    so = o.stats()
    for k in ("updates", "departures", "arrivals", "transitions", "lane_changes"):
        assert sum(res[r]["stats"][k] for r in range(world)) == so[k], k
