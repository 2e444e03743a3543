"""Per-CTA phase completion times at the peak of the bay workload (LPSIM_FLAG_TIMING)."""
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
    # grid size: try common sizes
    for gb in (444, 296, 592, 148, 888, 1184):
        try:
            bt = sim.lpsim_debug_block_times(gb)
            break
        except Exception:
            continue
    a = bt[:, 0] / n / 1e3
    c = bt[:, 1] / n / 1e3
    print("hour", hour, "on_road", s["on_road"], "us/step", 1e3 * s["step_ms"] / n, "phases", [x / n / 1e3 for x in s["phase_ns"]])
    for name, col in (("A", 2), ("C", 3)):
        st = bt[:, col].astype(np.int64)
        st = st[st > 0]
        print("  phase %s start skew over CTAs (last step, ns): p50 %d p90 %d max %d" % (
            name, np.percentile(st - st.min(), 50), np.percentile(st - st.min(), 90), (st - st.min()).max()))
    for name, x in (("A", a), ("C", c)):
        q = np.percentile(x, [0, 50, 90, 99, 100])
        print("  phase", name, "per-CTA us: min %.2f p50 %.2f p90 %.2f p99 %.2f max %.2f" % tuple(q),
              "slowest CTAs", np.argsort(-x)[:8].tolist())
    sim.close()
