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
    """SM clocks / throttle reasons sampled DURING the timed region (B200_PROFILING.md's clocks line),
    through NVML (the library nvidia-smi reads) in a host thread every 20 ms.  (r2 used a background
    `nvidia-smi -lms` whose block-buffered output was lost when it was terminated: 0 samples.)"""

    NAMES = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
             ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
             ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
             ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.thread = None
        self.samples = []
        self.err = None

    def _handle(self, nv):
        try:  # the CUDA device's PCI bus id (CUDA_VISIBLE_DEVICES may renumber devices)
            import torch

            p = torch.cuda.get_device_properties(self.gpu)
            bus = "%08x:%02x:%02x.0" % (p.pci_domain_id, p.pci_bus_id, p.pci_device_id)
            return nv.nvmlDeviceGetHandleByPciBusId_v2(bus)
        except Exception:
            return nv.nvmlDeviceGetHandleByIndex(self.gpu)

    def start(self):
        import threading

        try:
            import pynvml as nv

            nv.nvmlInit()
            h = self._handle(nv)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
        except Exception as e:  # no NVML: recorded, not silently empty
            self.err = "nvml unavailable: %s" % e
            return
        self.stop_evt = threading.Event()

        def run():
            while not self.stop_evt.is_set():
                try:
                    sm = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                    r = int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))
                    self.samples.append((sm, r))
                except Exception as e:
                    self.err = str(e)
                self.stop_evt.wait(0.02)

        self.nv = nv
        self.thread = threading.Thread(target=run, daemon=True)
        self.thread.start()

    def stop(self):
        if not self.thread:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err or "not started"], "samples": 0}
        self.stop_evt.set()
        self.thread.join()
        reasons = set()
        for n, attr in self.NAMES:
            bit = getattr(self.nv, attr, None)
            if bit is not None and any(r & bit for _, r in self.samples):
                reasons.add(n)
        sm = [s for s, _ in self.samples]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_min_mhz": min(sm) if sm else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(reasons), "samples": len(sm), "source": "NVML, 20 ms"}


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


def run_oracle_sample(g, d, peak_s, window_s, warmup, steps, openmp):
    """The reference arm: the oracle as it stands on the bounded peak sample; a ramp to a loaded state
    (untimed), W warm-up steps, then exactly K timed steps (one step = one simulation timestep, as in
    our arm)."""
    import oracle

    s = peak_sample(g, d, peak_s, window_s)
    o = oracle.Oracle(g, openmp=openmp)
    o.load_demand(s["depart_s"], s["route_ptr"], s["route_edges"])
    ramp = int(window_s / 0.5)
    o.step(ramp + warmup)
    u0 = o.stats()["updates"]
    on_road = int(o.stats()["on_road"])
    t0 = time.perf_counter()
    o.step(steps)
    dt = time.perf_counter() - t0
    upd = o.stats()["updates"] - u0
    o.close()
    return {"value": upd / dt if dt > 0 else 0.0, "steps": steps, "updates": int(upd), "seconds": dt,
            "trips": int(s["depart_s"].shape[0]), "ramp_steps": ramp, "on_road": on_road}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_oracle_at_state(g, d, ck, budget_s, openmp):
    """CPU baseline at exactly the GPU window's load: the oracle (timing only — parity is the tests'
    job) put at the GPU's checkpoint of the window start (lo_set_state), then timed for budget_s."""
    import oracle

    o = oracle.Oracle(g, openmp=openmp)
    o.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
    o.set_state(ck["step"], ck["status"], ck["edge"], ck["lane"], ck["pos"], ck["v"], ck["cursor"],
                ck["arrival_step"])
    o.step(1)  # warm-up
    u0 = o.stats()["updates"]
    t0 = time.perf_counter()
    n = 0
    while time.perf_counter() - t0 < budget_s:
        o.step(1)
        n += 1
    dt = time.perf_counter() - t0
    upd = o.stats()["updates"] - u0
    on_road = int(o.stats()["on_road"])
    o.close()
    return {"value": upd / dt if dt > 0 else 0.0, "steps": n, "updates": int(upd), "seconds": dt, "on_road": on_road}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

PART_DESC = {"pilot": "weights = vehicles on the road at the window start, from a pilot run",
             "visits": "weights = route visits over the demand"}


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

    node_part = None
    if (world > 1 or args.parts > 1) and args.partition == "pilot":
        # balanced for the load of the timed window (pilot run to the window start);
        # deterministic, so every rank computes the same partition
        from paper_2406_08496_b200.multi import pilot_partition

        node_part = pilot_partition(g, d, max(world, args.parts), args.peak_s, device=dev)

    def make_sim():
        kw = dict(device=dev, stream=C_stream(stream))
        if node_part is not None:
            kw["node_part"] = node_part.ctypes.data
        if args.sort_every:
            kw["sort_every"] = args.sort_every
        if args.ablation != "none":  # §8(f) item 4: what the lowest-id rule / the IDM free term / a9 cost
            kw["flags"] = {"racy": pkg.FLAG_RACY, "vfree": pkg.FLAG_VFREE, "nosort": pkg.FLAG_NO_SORT}[args.ablation]
        if world > 1:
            kw.update(rank=rank, world=world)
        elif args.parts > 1:  # K partitions in one process on one GPU (the multi-GPU exchange, in-process)
            kw["num_parts"] = args.parts
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
    if world == 1 and not args.no_cpu_baseline:
        out["checkpoint"] = sim.checkpoint()  # the window start, for the CPU baseline at the same load
    if os.environ.get("LPSIM_EXP_FLAGS"):  # timing experiments of experiment builds (tools/ab.sh)
        sim.set_flags(int(os.environ["LPSIM_EXP_FLAGS"], 0))
    for _ in range(args.warmup):
        with torch.cuda.stream(stream):
            flush.zero_()
        sim.step(1)
    sampler = ClockSampler(dev)
    sampler.start()
    if world > 1:
        torch.distributed.barrier(gloo)
    torch.cuda.synchronize()
    # three timed windows (median): world == 1, K one-step calls each preceded by an L2 flush (the
    # cold step); world > 1, K steps per call after one flush, so that launch skew between the
    # processes does not enter the per-step time
    wins = []
    launches = 0
    torch.cuda.nvtx.range_push("timed")
    for _w in range(3):
        ms, upd = 0.0, 0
        if world == 1:
            for _ in range(args.steps):
                with torch.cuda.stream(stream):
                    flush.zero_()  # L2 flush between timed steps (256 MiB > 126 MB L2)
                u0 = sim.stats()["updates"]
                sim.step(1)
                st = sim.stats()
                ms += st["step_ms"]
                upd += st["updates"] - u0
                launches += st["kernel_launches"]
        else:
            with torch.cuda.stream(stream):
                flush.zero_()
            u0 = sim.stats()["updates"]
            sim.step(args.steps)
            st = sim.stats()
            ms += st["step_ms"]
            upd += st["updates"] - u0
            launches += st["kernel_launches"]
        wins.append((reduce_max([ms])[0], int(reduce_sum([float(upd)])[0])))  # max over ranks
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    t_sampler = time.time()
    wins.sort(key=lambda w: w[0] / max(1, w[1]))
    t_ms, updates = wins[1]  # the median window (per-update time)
    on_road = int(reduce_sum([float(s_ff["on_road"])])[0])
    out["window"] = {"ms_total": t_ms, "updates": updates, "launches": launches // 3, "on_road_at_start": on_road,
                     "ffwd_steps": ffwd, "ffwd_wall_s": round(ffwd_wall, 3),
                     "windows_ms_per_step": [w[0] / args.steps for w in wins]}
    extra = 0
    if world == 1:
        # the same one-step calls from a clean cold L2: the write flush, then a 256 MiB read, so the
        # dirty flush lines are written back before the step starts (what ncu's cache control does
        # before its kernel replays).  Reported beside the headline, which keeps the write flush alone.
        flush_r = torch.empty_like(flush)
        ms_c = 0.0
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
                flush_r.sum()
            sim.step(1)
            ms_c += sim.stats()["step_ms"]
        extra = args.steps
        out["window"]["clean_l2_ms_per_step"] = ms_c / args.steps
        del flush_r
    # a9: the dead entries arrivals and migrations leave until the next compaction, just before a sort
    sort_every = args.sort_every or 256
    k_now = ffwd + args.warmup + 3 * args.steps + extra
    to_sort = (sort_every - 1) - (k_now % sort_every)
    if to_sort > 0:
        sim.step(to_sort)
    st = sim.stats()
    out["dead_entries"] = {"soa_entries": int(reduce_sum([float(st["soa_entries"])])[0]),
                           "on_road": int(reduce_sum([float(st["on_road"])])[0]),
                           "steps_since_sort": sort_every - 1}
    # steady state (no flush): one sort period in one call (the sort's own device time is reported)
    torch.cuda.nvtx.range_push("steady")
    u0 = sim.stats()["updates"]
    sim.step(sort_every)
    torch.cuda.nvtx.range_pop()
    st = sim.stats()
    out["steady"] = {"ms": reduce_max([st["step_ms"]])[0], "steps": sort_every,
                     "updates": int(reduce_sum([float(st["updates"] - u0)])[0]),
                     "sort_ms": reduce_max([st["sort_ns"] / 1e6])[0]}
    # the clock record spans the timed windows and the steady segment; the GPU is kept stepping until
    # the sampler has 2 s of samples (nvidia-smi samples every 100 ms)
    while time.time() - t_sampler < 2.0:
        sim.step(1024)
    torch.cuda.synchronize()
    out["clocks"] = sampler.stop()
    if world > 1:
        # NVLink exchange per step: the migrants, their counts and the mirrored halo bytes are stored into
        # the peers' memory by phases A and C themselves; what remains is the step's one cross-GPU flag
        # barrier (count push + release/acquire over NVLink).  Device timers of the instrumented kernel,
        # one step per call, the distribution over the steps (max over ranks per step)
        sim.set_flags(pkg.FLAG_TIMING)
        ex = []
        for _ in range(args.steps):
            sim.step(1)
            ex.append(reduce_max([sim.stats()["exchange_ms"] * 1e3])[0])
        sim.set_flags(0)
        ex = np.array(ex)
        out["exchange"] = {"us_per_step_median": float(np.median(ex)), "us_per_step_p99": float(np.percentile(ex, 99)),
                           "us_per_step_mean": float(ex.mean()), "steps": int(ex.size),
                           "what": "cross-GPU barrier device time per step (max over ranks; the peer stores are "
                                   "inside phases A and C), instrumented kernel, no flush"}
    sim.close()
    del sim

    # ---- (2) full demand end to end through the public API (host arrays) ----
    if not args.no_full_run:
        torch.cuda.synchronize()
        h2d = sum(int(np.asarray(g[k]).nbytes) for k in ("row_ptr", "dst", "length_m", "lanes", "speed_limit_mps")) \
            + sum(int(d[k].nbytes) for k in ("depart_s", "route_ptr", "route_edges"))
        if world > 1:
            torch.distributed.barrier(gloo)
        os.environ["LPSIM_LOAD_TIMES"] = "1"  # the load's host / setup stage times on stderr (diagnostics)
        t0 = time.perf_counter()
        sim = make_sim()
        t_load = time.perf_counter() - t0
        os.environ.pop("LPSIM_LOAD_TIMES", None)
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
    ap.add_argument("--cpu-budget-s", type=float, default=20.0, help="oracle timing budget (split 1 core / all cores)")
    ap.add_argument("--parts", type=int, default=1, help="N=1 only: K partitions (multilevel) in one process "
                    "on one GPU, exchanging through the same direct-write path as K GPUs")
    ap.add_argument("--partition", default="pilot", choices=["pilot", "visits"],
                    help="K > 1: multilevel partition balanced for the window's load (a pilot run to the window "
                         "start) or the built-in route-visit weights (P:L457)")
    ap.add_argument("--sort-every", type=int, default=0, help="locality sort period (a9); 0 = the library default")
    ap.add_argument("--ablation", default="none", choices=["none", "racy", "vfree", "nosort"],
                    help="racy: first-claimer-wins claims (P:L250); vfree: literal v <- v_free (P:L320); "
                         "nosort: no a9 locality sort (compaction only)")
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
        r = run_oracle_sample(g, d, args.peak_s, 600.0, args.warmup, args.steps, openmp=True)
        line = {"impl": "reference", "metric": METRIC, "value": r["value"], "unit": "updates/s", "n_gpus": args.gpus,
                "steps": r["steps"], "warmup": args.warmup, "ms_per_step": 1e3 * r["seconds"] / max(1, r["steps"]),
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic",
                "config": dict(workload, parallelism="cpu oracle (OpenMP build), %s threads" %
                               os.environ.get("OMP_NUM_THREADS", cores)),
                "cpu_baseline": {"value": r["value"], "unit": "updates/s", "cores": cores, "kind": "oracle",
                                 "cpu_model": cpu_model(),
                                 "sample": "trips departing in the 10 min after t=%.0fs (%d trips) shifted to t=0, "
                                           "%d ramp steps + %d warm-up steps untimed (%d on the road), then %d steps "
                                           "timed (%.2f s)" % (args.peak_s, r["trips"], r["ramp_steps"], args.warmup,
                                                              r["on_road"], r["steps"], r["seconds"])},
                "e2e": {"value": r["value"], "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return 0

    out = run_ours(args, g, d, meta, rank, world, local_rank)
    w = out["window"]
    st = out["steady"]
    # every simulated step pays 1/sort_every of an a9 sort (the cold windows contain none): its measured
    # device time is added per step
    sort_every = args.sort_every or 256
    sort_ms_per_step = st["sort_ms"] / sort_every
    ms_per_step = w["ms_total"] / args.steps + sort_ms_per_step
    value = w["updates"] / (ms_per_step * args.steps / 1e3)
    pk = peaks()
    hbm_peak = pk["hbm_gbs"] if pk else 6650.0
    # roofline of the dominant kernel (k_run: the fused step): algorithmic bytes per launch over the
    # launch's CUDA-event time
    upd_per_step_rank = w["updates"] / args.steps / max(1, world)
    kernel_ms = w["ms_total"] / args.steps
    achieved = upd_per_step_rank * ALG_BYTES_PER_UPDATE / (kernel_ms / 1e3) / 1e9
    traffic, traffic_src = None, None
    tp = os.path.join(ROOT, "profiles", "k_run_dram_bytes_per_update.json")
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp))
            traffic, traffic_src = tj.get("dram_bytes_per_launch"), tj.get("source")
        except Exception:
            traffic = None
    line = {
        "metric": METRIC, "value": value, "unit": "updates/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": dict(workload, parallelism=("single partition" if args.parts == 1 else
                                              "%d partitions (multilevel k-way, %s) in one process on one GPU" % (args.parts, PART_DESC[args.partition]))
                       if world == 1 else
                       "%d partitions (multilevel k-way, %s), one per GPU, NVLink peer-memory exchange" % (world, PART_DESC[args.partition]),
                       timing=("median of 3 windows of %d one-step calls, L2 flushed before each; + the amortized "
                               "a9 sort (%.3f ms every %d steps)" % (args.steps, st["sort_ms"], sort_every)) if world == 1 else
                       ("median of 3 windows of %d steps in one call each, L2 flushed before each; + the amortized "
                        "a9 sort" % args.steps)),
        "gpu_launches": w["launches"],
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic, "traffic_source": traffic_src,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)" if pk else "fallback 6.65 TB/s",
                     "alg_bytes_per_update": ALG_BYTES_PER_UPDATE, "kernel": "k_run (fused step)",
                     "kernel_ms_per_launch": kernel_ms},
        "clocks": out["clocks"],
        "steady_state": {"ms_per_step": st["ms"] / st["steps"], "steps": st["steps"], "sort_ms": st["sort_ms"],
                         "updates_per_s": st["updates"] / (st["ms"] / 1e3),
                         "roofline_frac": st["updates"] / max(1, world) * ALG_BYTES_PER_UPDATE / (st["ms"] / 1e3) / 1e9
                         / hbm_peak,
                         "note": "one sort period in one call, no flush (how a full run executes), sort included; "
                                 "roofline_frac = the same algorithmic bytes over this time, same peak"},
        "window": {"on_road_at_start": w["on_road_at_start"], "ffwd_steps": w["ffwd_steps"],
                   "windows_ms_per_step": w["windows_ms_per_step"],
                   "clean_l2_ms_per_step": w.get("clean_l2_ms_per_step"),
                   "clean_l2_note": "one-step calls after the write flush and a 256 MiB read (dirty flush lines "
                                    "written back before the step, as ncu's cache control does); not the headline"},
        "dead_entries": dict(out["dead_entries"], share=1.0 - out["dead_entries"]["on_road"] /
                             max(1, out["dead_entries"]["soa_entries"])),
        "exchange": out.get("exchange", {"us_per_step_median": 0.0, "what": "single partition: no exchange"}),
    }
    if world > 1:
        line["comm"] = {"data_plane": "CUDA IPC peer memory: the step kernel stores migrants and entry-halo bytes "
                                      "into the peers' HBM over NVLink, one in-kernel flag barrier per step",
                        "process_group": "NCCL group initialised for the launch contract; it carries no data "
                                         "(a gloo group bootstraps the IPC records and combines the results)"}
    if "full" in out:
        f = out["full"]
        line["full_run"] = {"wall_s": f["wall_s"], "device_s": f["device_s"], "load_s": f["load_s"],
                            "steps": f["steps"], "updates": f["updates"], "arrived": f["arrived"], "trips": f["trips"],
                            "mean_travel_time_s": f["mean_travel_time_s"]}
        line["e2e"] = {"value": f["updates"] / f["wall_s"], "unit": "updates/s",
                       "h2d_bytes_per_step": f["h2d_bytes"] / f["steps"], "d2h_bytes_per_step": f["d2h_bytes"] / f["steps"],
                       "wall_s": f["wall_s"], "what": "create+load_demand+step until drained+results from host arrays"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ck = out["checkpoint"]
        r1 = run_oracle_at_state(g, d, ck, args.cpu_budget_s / 2, openmp=False)
        rn = run_oracle_at_state(g, d, ck, args.cpu_budget_s / 2, openmp=True)
        line["cpu_baseline"] = {"value": rn["value"], "unit": "updates/s", "cores": cores, "kind": "oracle",
                                "sample": "the oracle (OpenMP build, OMP_NUM_THREADS=%s) put at the GPU's checkpoint of "
                                          "the window start (t=%.0fs, %d on road: the same load; timing only), %d steps "
                                          "(%.1f s)" % (os.environ.get("OMP_NUM_THREADS", cores), args.peak_s,
                                                        rn["on_road"], rn["steps"], rn["seconds"]),
                                "one_core": {"value": r1["value"], "cores": 1, "steps": r1["steps"],
                                             "seconds": r1["seconds"]},
                                "cpu_model": cpu_model(), "host_cores_available": cores}
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        import torch

        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
