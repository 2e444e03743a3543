"""Diagnostics of a synthetic workload's traffic state (not part of the bench).

Runs the full demand on the GPU and prints an hourly timeline (on-road,
arrived, departures); optionally dumps the lane map at given hours so the
jammed edges can be inspected offline.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="bay")
    ap.add_argument("--trips", type=int, default=None)
    ap.add_argument("--hours", type=float, default=24.0)
    ap.add_argument("--dump-at", type=float, nargs="*", default=[])
    ap.add_argument("--out", default="gpurun_out")
    ap.add_argument("--set", nargs="*", default=[], help="generator overrides key=value")
    a = ap.parse_args()
    from paper_2406_08496_b200 import Simulation
    from workloads import make_workload

    ov = {kv.split("=")[0]: float(kv.split("=")[1]) for kv in a.set}
    for k in ("fwy_every", "fwy_skip", "zones"):
        if k in ov:
            ov[k] = int(ov[k])
    g, d, meta = make_workload(a.workload, trips=a.trips, cache_dir="/tmp/lpsim_cache", **ov)
    print(json.dumps({k: v for k, v in meta.items() if k not in ("dep",)}), flush=True)
    sim = Simulation(g)
    sim.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
    rows = []
    steps_per_h = 7200
    t0 = time.time()
    for h in range(int(a.hours)):
        sim.step(steps_per_h)
        s = sim.stats()
        rows.append(dict(hour=h + 1, on_road=s["on_road"], waiting=s["waiting"], finished=s["finished"],
                         ms_per_step=s["step_ms"] / steps_per_h))
        print(json.dumps(rows[-1]), flush=True)
        if (h + 1) in [int(x) for x in a.dump_at]:
            m = sim.lane_map()
            np.savez_compressed(os.path.join(a.out, "lanemap_%s_%dk_h%d.npz" % (a.workload, (a.trips or meta["trips"]) // 1000, h + 1)), m=m)
        if s["on_road"] == 0 and s["waiting"] == 0:
            break
    arr, t, dist = sim.results()
    ok = arr >= 0
    tt = t[ok] - d["depart_s"][ok]
    print(json.dumps(dict(trips=int(arr.shape[0]), arrived=int(ok.sum()), mean_tt_s=float(tt.mean()) if ok.any() else None,
                          p50_tt=float(np.median(tt)) if ok.any() else None, p95_tt=float(np.percentile(tt, 95)) if ok.any() else None,
                          mean_free_km=float(dist[ok].mean() / 1000) if ok.any() else None, wall_s=time.time() - t0)))


if __name__ == "__main__":
    main()
