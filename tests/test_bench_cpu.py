"""bench.py host logic (no GPU): the clock sampler degrades to an explicit reason, the reference arm
times exactly K steps of the oracle after W warm-up steps on its bounded sample."""
import importlib.util
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_clock_sampler_without_gpu_reports_why():
    b = _bench()
    s = b.ClockSampler(0)
    s.start()
    r = s.stop()
    assert set(r) >= {"sm_mhz", "sm_max_mhz", "reasons", "samples"}
    if r["samples"] == 0:  # no NVML device here: the line says so instead of an empty record
        assert r["reasons"] and isinstance(r["reasons"][0], str)


def test_reference_arm_times_exactly_k_steps():
    from workloads import make_workload

    b = _bench()
    g, d, meta = make_workload("grid4b", cache_dir="/tmp/lpsim_cache")
    r = b.run_oracle_sample(g, d, 0.0, 120.0, warmup=3, steps=7, openmp=False)
    assert r["steps"] == 7
    assert r["ramp_steps"] == 240
    assert r["updates"] > 0 and r["value"] > 0
    # the sample is the trips departing in the window, shifted to t = 0
    s = b.peak_sample(g, d, 0.0, 120.0)
    assert s["depart_s"].shape[0] == r["trips"]
    assert np.all(s["depart_s"] >= 0.0) and np.all(s["depart_s"] < 120.0)
