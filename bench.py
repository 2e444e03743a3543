#!/usr/bin/env python
"""Benchmark of the B200-native LPSim per-timestep vehicle update.

Metric (BASELINE.json): vehicle-updates/s and full-demand wall time; % of the
HBM roofline.  One bench "step" = one simulation timestep k -> k+1 = one pass
of every §8(a) row over all active vehicles of the workload.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload bay9m] [--trips T] [--peak-s 28800] [--no-full-run]

Default workload: C4 "bay9m" (synthetic Bay-Area-shaped graph, 9,008,766 trips
over 12 h, P:L63 — BASELINE.json configs[3], the one configuration the metric
is quoted on at 1/2/4/8 GPUs and the north_star target; it fits one B200).
`--workload bay` runs C3 (2.82M trips, the paper's single-GPU case).  The timed
window starts at the AM peak (t = 8:00 h, reached by simulating from t = 0);
each timed step is preceded by an L2 flush (a 256 MiB write) and timed with
CUDA events on the launching stream.  `e2e` runs the whole demand through the
public API from host arrays (create -> load_demand -> step until drained ->
results), wall-clock, host<->device copies included.

--impl reference: the CPU oracle (the base contract's reference arm for this
tier), timed on a bounded sample of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

ALG_BYTES_PER_UPDATE = 64  # SURVEY §8(d) algorithmic bytes per vehicle-update
METRIC = "vehicle-updates/s"
CACHE = os.environ.get("LPSIM_CACHE", "/tmp/lpsim_cache")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region (B200_PROFILING.md)."""

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = "/tmp/lpsim_clocks_%d_%d.csv" % (os.getpid(), gpu_index)

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def load_workload(name, trips, rank):
    from workloads import make_workload

    t0 = time.time()
    g, d, meta = make_workload(name, trips=trips, cache_dir=CACHE)
    meta["gen_wall_s"] = round(time.time() - t0, 2)
    return g, d, meta


# ---------------------------------------------------------------------------
# reference arm / cpu baseline: the oracle on a bounded sample
# ---------------------------------------------------------------------------

def peak_sample(g, d, peak_s, window_s):
    """Trips departing in [peak_s, peak_s + window_s), shifted to t = 0."""
    sel = np.nonzero((d["depart_s"] >= peak_s) & (d["depart_s"] < peak_s + window_s))[0]
    rl = np.diff(d["route_ptr"])[sel]
    rp = np.zeros(sel.shape[0] + 1, np.int64)
    np.cumsum(rl, out=rp[1:])
    idx = np.concatenate([np.arange(d["route_ptr"][i], d["route_ptr"][i + 1]) for i in sel]) if sel.size else \
        np.zeros(0, np.int64)
    return {"depart_s": d["depart_s"][sel] - peak_s, "route_ptr": rp, "route_edges": d["route_edges"][idx]}


def run_oracle_sample(g, d, peak_s, window_s, warmup, steps, budget_s):
    import oracle

    s = peak_sample(g, d, peak_s, window_s)
    o = oracle.Oracle(g)
    o.load_demand(s["depart_s"], s["route_ptr"], s["route_edges"])
    # bring the sample to a loaded state (untimed), then time steps until budget or `steps`
    ramp = int(window_s / 0.5)
    o.step(ramp + warmup)
    u0 = o.stats()["updates"]
    t0 = time.perf_counter()
    n = 0
    while n < steps or (time.perf_counter() - t0) < min(10.0, budget_s):  # >= 10 s of timed oracle work
        o.step(1)
        n += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    upd = o.stats()["updates"] - u0
    return {"value": upd / dt if dt > 0 else 0.0, "steps": n, "updates": int(upd), "seconds": dt,
            "trips": int(s["depart_s"].shape[0]), "ramp_steps": ramp}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours(args, g, d, meta, rank, world, local_rank):
    """world == 1: the whole workload on one GPU.  world > 1: one partition per
    GPU (route-weighted multilevel k-way partition, §8(e)), migrants and entry halos exchanged by the
    step kernel over NVLink peer memory; strong scaling (fixed workload)."""
    import torch

    import paper_2406_08496_b200 as pkg
    from paper_2406_08496_b200.multi import attach_peers

    # LPSIM_BENCH_SAME_GPU=1: every rank on device 0 (time-sliced), to exercise the multi-rank path
    # (IPC peer memory, in-kernel exchange, reductions, the JSON line) on a one-GPU box
    dev = 0 if os.environ.get("LPSIM_BENCH_SAME_GPU") else local_rank
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream(device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    gloo = None
    if world > 1:
        import torch.distributed as dist

        gloo = dist.new_group(backend="gloo")
    out = {}

    def make_sim():
        kw = dict(device=dev, stream=C_stream(stream))
        if args.sort_every:
            kw["sort_every"] = args.sort_every
        if args.ablation != "none":  # §8(f) item 4: what the lowest-id rule / the IDM free term cost
            kw["flags"] = pkg.FLAG_RACY if args.ablation == "racy" else pkg.FLAG_VFREE
        if world > 1:
            kw.update(rank=rank, world=world)
        sim = pkg.Simulation(g, **kw)
        sim.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
        if world > 1:
            attach_peers(sim, gloo)
            torch.distributed.barrier(gloo)
        return sim

    def reduce_sum(vals):
        if world == 1:
            return vals
        t = torch.tensor(vals, dtype=torch.float64)
        torch.distributed.all_reduce(t, group=gloo)
        return t.tolist()

    def reduce_max(vals):
        if world == 1:
            return vals
        t = torch.tensor(vals, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX, group=gloo)
        return t.tolist()

    # ---- (1) windowed measurement at the peak, state resident in HBM ----
    sim = make_sim()
    ffwd = int(args.peak_s / 0.5)
    t0 = time.time()
    sim.step(ffwd)
    torch.cuda.synchronize()
    ffwd_wall = time.time() - t0
    s_ff = sim.stats()
    if os.environ.get("LPSIM_EXP_FLAGS"):  # timing experiments of experiment builds (tools/ab.sh)
        sim.set_flags(int(os.environ["LPSIM_EXP_FLAGS"], 0))
    for _ in range(args.warmup):
        with torch.cuda.stream(stream):
            flush.zero_()
        sim.step(1)
    step_ms, updates, launches = [], 0, 0
    sampler = ClockSampler(dev)
    sampler.start()
    if world > 1:
        torch.distributed.barrier(gloo)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("timed")
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()  # L2 flush between timed steps (256 MiB > 126 MB L2)
        u0 = sim.stats()["updates"]
        sim.step(1)
        s = sim.stats()
        step_ms.append(s["step_ms"])
        updates += s["updates"] - u0
        launches += s["kernel_launches"]
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    t_ms = reduce_max([float(sum(step_ms))])[0]  # max over ranks
    updates = int(reduce_sum([float(updates)])[0])
    on_road = int(reduce_sum([float(s_ff["on_road"])])[0])
    out["window"] = {"ms_total": t_ms, "updates": updates, "launches": launches, "on_road_at_start": on_road,
                     "ffwd_steps": ffwd, "ffwd_wall_s": round(ffwd_wall, 3)}
    out["clocks"] = clocks
    # steady state (no flush): K steps in one call
    torch.cuda.nvtx.range_push("steady")
    sim.step(args.steps)
    torch.cuda.nvtx.range_pop()
    out["steady"] = {"ms": reduce_max([sim.stats()["step_ms"]])[0], "steps": args.steps}
    if world > 1:
        # NVLink exchange per step (phase X: migrant ingest + entry-halo publish + the grid and
        # cross-GPU flag barriers), device timers of the instrumented kernel, separate K-step window
        sim.set_flags(pkg.FLAG_TIMING)
        sim.step(args.steps)
        st = sim.stats()
        sim.set_flags(0)
        ph = [float(x) / 1e3 / args.steps for x in st["phase_ns"]]
        out["exchange"] = {"us_per_step": reduce_max([st["exchange_ms"] * 1e3 / args.steps])[0],
                           "phase_us_per_step": {"move": reduce_max([ph[0]])[0], "resolve": reduce_max([ph[1]])[0],
                                                 "exchange": reduce_max([ph[2]])[0]},
                           "step_us_instrumented": reduce_max([st["step_ms"] * 1e3 / args.steps])[0],
                           "what": "phase X device time per step (max over ranks), instrumented kernel, no flush"}
    sim.close()
    del sim

    # ---- (2) full demand end to end through the public API (host arrays) ----
    if not args.no_full_run:
        torch.cuda.synchronize()
        h2d = sum(int(np.asarray(g[k]).nbytes) for k in ("row_ptr", "dst", "length_m", "lanes", "speed_limit_mps")) \
            + sum(int(d[k].nbytes) for k in ("depart_s", "route_ptr", "route_edges"))
        if world > 1:
            torch.distributed.barrier(gloo)
        t0 = time.perf_counter()
        sim = make_sim()
        t_load = time.perf_counter() - t0
        steps = 0
        dev_ms = 0.0
        horizon = int(meta["horizon_s"] / 0.5)
        chunk = 3600
        while True:
            sim.step(chunk)
            steps += chunk
            st = sim.stats()
            dev_ms += st["step_ms"]
            left = meta["trips"] - reduce_sum([float(st["arrivals"])])[0]  # every trip arrives on one rank
            if steps >= horizon and left == 0:
                break
            if steps >= 2 * horizon:
                break
        a, tt_, dist = sim.results()
        if world > 1:
            from paper_2406_08496_b200.multi import combine_results

            a, dist = combine_results(a, dist, gloo)
            tt_ = np.where(a >= 0, a * 0.5, -1.0)
        wall = time.perf_counter() - t0
        d2h = a.nbytes + tt_.nbytes + dist.nbytes
        st = sim.stats()
        upd = int(reduce_sum([float(st["updates"])])[0])
        wall = reduce_max([wall])[0]
        dev_s = reduce_max([dev_ms / 1e3])[0]
        out["full"] = {"wall_s": wall, "load_s": t_load, "steps": steps, "device_s": dev_s,
                       "updates": upd, "arrived": int((a >= 0).sum()), "trips": int(a.shape[0]),
                       "h2d_bytes": h2d, "d2h_bytes": d2h,
                       "mean_travel_time_s": float(np.mean(tt_[a >= 0] - d["depart_s"][a >= 0])) if (a >= 0).any() else None}
        sim.close()
    return out


def C_stream(stream):
    return stream.cuda_stream


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=128)  # one sort period (a9) in the window
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="bay9m")
    ap.add_argument("--trips", type=int, default=None)
    ap.add_argument("--peak-s", type=float, default=8 * 3600.0)
    ap.add_argument("--no-full-run", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=20.0)
    ap.add_argument("--sort-every", type=int, default=0, help="locality sort period (a9); 0 = the library default")
    ap.add_argument("--ablation", default="none", choices=["none", "racy", "vfree"],
                    help="racy: first-claimer-wins claims (P:L250); vfree: literal v <- v_free (P:L320)")
    args = ap.parse_args()
    rank, world, local_rank = dist_env()
    if args.impl == "reference" and rank != 0:
        return 0  # the oracle reference runs on rank 0 only
    if world > 1 and args.impl == "ours":
        import torch

        if os.environ.get("LPSIM_BENCH_SAME_GPU"):
            torch.cuda.set_device(0)
            torch.distributed.init_process_group("gloo")
        else:
            torch.cuda.set_device(local_rank)
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    g, d, meta = load_workload(args.workload, args.trips, rank)
    workload = {"workload": "%s (%s)" % (args.workload, meta.get("kind")), "nodes": meta["nodes"],
                "edges": meta["edges"], "cells": meta["cells"], "trips": meta["trips"],
                "horizon_s": meta["horizon_s"], "seed": meta["seed"], "window_start_s": args.peak_s,
                "l2": "flushed before every timed step (256 MiB write)"}
    if args.ablation != "none":
        workload["ablation"] = args.ablation
    cores = os.cpu_count()

    if args.impl == "reference":
        r = run_oracle_sample(g, d, args.peak_s, 600.0, args.warmup, args.steps, budget_s=max(5.0, args.cpu_budget_s))
        line = {"impl": "reference", "metric": METRIC, "value": r["value"], "unit": "updates/s", "n_gpus": args.gpus,
                "steps": r["steps"], "warmup": args.warmup, "ms_per_step": 1e3 * r["seconds"] / max(1, r["steps"]),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": dict(workload, parallelism="cpu oracle, 1 thread"),
                "cpu_baseline": {"value": r["value"], "unit": "updates/s", "cores": 1, "kind": "oracle",
                                 "sample": "trips departing in the 10 min after t=%.0fs (%d trips) shifted to t=0, "
                                           "%d ramp steps untimed, then %d steps timed" %
                                           (args.peak_s, r["trips"], r["ramp_steps"], r["steps"])},
                "e2e": {"value": r["value"], "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return 0

    out = run_ours(args, g, d, meta, rank, world, local_rank)
    w = out["window"]
    ms_per_step = w["ms_total"] / args.steps
    value = w["updates"] / (w["ms_total"] / 1e3)
    pk = peaks()
    hbm_peak = pk["hbm_gbs"] if pk else 6650.0
    # roofline of the dominant kernel (k_run: the fused step) — DESIGN.md §8
    upd_per_step_rank = w["updates"] / args.steps / max(1, world)
    achieved = upd_per_step_rank * ALG_BYTES_PER_UPDATE / (ms_per_step / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "k_run_dram_bytes_per_update.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    line = {
        "metric": METRIC, "value": value, "unit": "updates/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": dict(workload, parallelism="single partition" if world == 1 else
                       "%d partitions (route-weighted multilevel k-way), one per GPU, NVLink peer-memory exchange" % world),
        "gpu_launches": w["launches"],
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)" if pk else "fallback 6.65 TB/s",
                     "alg_bytes_per_update": ALG_BYTES_PER_UPDATE, "kernel": "k_run (fused step)"},
        "clocks": out["clocks"],
        "steady_state": {"ms_per_step": out["steady"]["ms"] / args.steps, "note": "same K steps in one call, no flush"},
        "window": {"on_road_at_start": w["on_road_at_start"], "ffwd_steps": w["ffwd_steps"]},
        "exchange": out.get("exchange", {"us_per_step": 0.0, "what": "single partition: no exchange"}),
    }
    if "full" in out:
        f = out["full"]
        line["full_run"] = {"wall_s": f["wall_s"], "device_s": f["device_s"], "load_s": f["load_s"],
                            "steps": f["steps"], "updates": f["updates"], "arrived": f["arrived"], "trips": f["trips"],
                            "mean_travel_time_s": f["mean_travel_time_s"]}
        line["e2e"] = {"value": f["updates"] / f["wall_s"], "unit": "updates/s",
                       "h2d_bytes_per_step": f["h2d_bytes"] / f["steps"], "d2h_bytes_per_step": f["d2h_bytes"] / f["steps"],
                       "wall_s": f["wall_s"], "what": "create+load_demand+step until drained+results from host arrays"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r = run_oracle_sample(g, d, args.peak_s, 600.0, 0, 1, budget_s=args.cpu_budget_s)
        line["cpu_baseline"] = {"value": r["value"], "unit": "updates/s", "cores": 1, "kind": "oracle",
                                "sample": "trips departing in the 10 min after t=%.0fs (%d trips) shifted to t=0; "
                                          "%d ramp steps untimed, then %d steps (%.1f s) timed" %
                                          (args.peak_s, r["trips"], r["ramp_steps"], r["steps"], r["seconds"]),
                                "host_cores_available": cores}
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        import torch

        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
