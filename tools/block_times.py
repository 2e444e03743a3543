"""Per-CTA phase and barrier times at two points of a workload (LPSIM_FLAG_TIMING).

For each phase: start skew over CTAs, per-CTA work (phase start -> slowest
warp done), barrier arrival spread, and the barrier's own latency (last
arrival -> first exit of the next phase).
"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_08496_b200 import FLAG_TIMING, Simulation
from workloads import make_workload

g, d, meta = make_workload(sys.argv[1] if len(sys.argv) > 1 else "bay", cache_dir="/tmp/lpsim_cache")
for hour in (1, 8):
    sim = Simulation(g, flags=FLAG_TIMING)
    sim.load_demand(d["depart_s"], d["route_ptr"], d["route_edges"])
    sim.step(hour * 7200 - 256)
    sim.step(256)
    s = sim.stats()
    n = 256
    for gb in (444, 296, 592, 148, 888, 1184):
        try:
            bt = sim.lpsim_debug_block_times(gb).astype(np.int64)
            break
        except Exception:
            continue
    print("hour", hour, "on_road", s["on_road"], "us/step", 1e3 * s["step_ms"] / n,
          "phases", [x / n / 1e3 for x in s["phase_ns"]], "grid", gb)
    t0 = bt[:, 2].min()
    for name, w, st, arr, wait, nxt in (("A", 0, 2, 4, 6, 3), ("C", 1, 3, 5, 7, None)):
        x = bt[:, w] / n / 1e3
        q = np.percentile(x, [0, 50, 90, 99, 100])
        starts = bt[:, st] - bt[:, st].min()
        arrivals = bt[:, arr]
        print("  phase %s (last step, ns rel. to first A start): start p50 %d max %d | arrival p50 %d max %d" % (
            name, np.median(bt[:, st] - t0), (bt[:, st] - t0).max(), np.median(arrivals - t0), (arrivals - t0).max()))
        if nxt is not None:
            print("    barrier after %s: last arrival -> first / median next-phase start: %d / %d ns" % (
                name, bt[:, nxt].min() - arrivals.max(), np.median(bt[:, nxt]) - arrivals.max()))
        late = np.argsort(-arrivals)[:6]
        print("    latest arrivals (cta: start/work end/arrival ns, chunk rounds):",
              ", ".join("%d: %d/%d/%d r%d" % (b, bt[b, st] - t0, bt[b, 8 + w] - t0, arrivals[b] - t0, bt[b, 10])
                        for b in late))
        if name == "C":
            dep = (bt[:, 18] & 0xFFFFFFFF) / n
            clm = (bt[:, 18] >> 32) / n
            rel = bt[:, 19] / n
            print("    per step: departures / claimed positions / relisted in the CTA's admit chunks — slowest CTAs:",
                  ", ".join("%d: %.1f / %.1f / %.1f" % (b, dep[b], clm[b], rel[b]) for b in np.argsort(bt[:, wait])[:4]),
                  "| median CTA: %.1f / %.1f / %.1f" % (np.median(dep), np.median(clm), np.median(rel)))
            print("    slowest CTAs' claims end / departures end, us (mean over steps):",
                  ", ".join("%d: %.2f / %.2f" % (b, bt[b, 14] / n / 1e3, bt[b, 15] / n / 1e3)
                            for b in np.argsort(bt[:, wait])[:4]))
        lw = np.argsort(bt[:, wait])[:6]
        print("    least total barrier wait (most often late):",
              ", ".join("%d: %.2f us" % (b, bt[b, wait] / n / 1e3) for b in lw))
        subs = (("probe in", 16), ("longitudinal", 17), ("first move", 11), ("vehicles end", 12),
                ("admit end", 13)) if name == "A" else \
            (("claims end", 14), ("departures end", 15))
        if name == "C":
            for b in np.argsort(bt[:, wait])[:4]:
                print("    CTA %d warp 0 admit chunk, us: position in %.2f, claim words %.2f, successors %.2f, written %.2f" % (
                    (b,) + tuple(bt[b, c] / n / 1e3 for c in (20, 21, 22, 23))))
        print("    thread-0 milestones from phase start, us (p50 / p90 / max over CTAs):",
              "; ".join("%s %.2f / %.2f / %.2f" % ((lab,) + tuple(np.percentile(bt[:, c] / n / 1e3, [50, 90, 100])))
                        for lab, c in subs))
        print("    per-CTA work us: min %.2f p50 %.2f p90 %.2f p99 %.2f max %.2f" % tuple(q),
              "slowest CTAs", np.argsort(-x)[:6].tolist(),
              "| mean barrier wait us %.2f" % (bt[:, wait].mean() / n / 1e3))
    sim.close()
