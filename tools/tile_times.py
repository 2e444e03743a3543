"""Per-tile timing of the step kernel at a chosen time of the simulated day.

Runs the workload to --at-s (untimed), then --steps steps with LPSIM_FLAG_TIMING and prints, over the
tiles, the distribution of the time per step spent waiting for neighbour tiles, moving and resolving,
and of the records per tile; the slowest tiles with their loads.  (Diagnostics for DESIGN.md §12.)

  python tools/tile_times.py [--workload bay9m] [--at-s 28800] [--steps 64]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="bay9m")
    ap.add_argument("--trips", type=int, default=None)
    ap.add_argument("--at-s", type=float, default=8 * 3600.0)
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    import paper_2406_08496_b200 as pkg
    from workloads import make_workload

    g, d, meta = make_workload(args.workload, trips=args.trips, cache_dir=os.environ.get("LPSIM_CACHE", "/tmp/lpsim_cache"))
    sim = pkg.Simulation(g, flags=0)
    sim.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
    sim.step(int(args.at_s / 0.5))
    s0 = sim.stats()
    sim.step(args.steps)
    steady_ms = sim.stats()["step_ms"]
    tiles = int(sim.stats()["tiles"])
    sim.lpsim_set_flags(pkg.FLAG_TIMING)
    sim.step(args.steps)
    st = sim.stats()
    bt = sim.lpsim_debug_block_times(tiles).astype(np.float64)
    n = max(1.0, float(args.steps))
    wait, move, res = bt[:, 0] / n / 1e3, bt[:, 1] / n / 1e3, bt[:, 2] / n / 1e3
    recs, nnb, cap = bt[:, 4], bt[:, 5], bt[:, 6]

    def q(x):
        return {"min": float(x.min()), "p50": float(np.median(x)), "p90": float(np.percentile(x, 90)),
                "max": float(x.max()), "mean": float(x.mean())}

    out = {"workload": args.workload, "at_s": args.at_s, "on_road": int(s0["on_road"]), "tiles": tiles,
           "steady_us_per_step": steady_ms * 1e3 / args.steps,
           "instrumented_us_per_step": st["step_ms"] * 1e3 / args.steps,
           "wait_us": q(wait), "move_us": q(move), "resolve_us": q(res), "records": q(recs), "neighbours": q(nnb)}
    busy = move + res
    top = np.argsort(-busy)[:8]
    out["slowest_tiles"] = [{"tile": int(t), "move_us": float(move[t]), "resolve_us": float(res[t]),
                             "wait_us": float(wait[t]), "records": int(recs[t]), "neighbours": int(nnb[t])}
                            for t in top]
    out["corr_busy_records"] = float(np.corrcoef(busy, recs)[0, 1]) if tiles > 2 else None
    print(json.dumps(out, indent=1))
    if args.json:
        json.dump(out, open(args.json, "w"), indent=1)


if __name__ == "__main__":
    main()
