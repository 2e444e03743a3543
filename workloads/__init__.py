"""Seeded synthetic workloads (road graphs + routed OD demand).

This package is the ONLY code shared by the oracle side and the CUDA side: it
produces inputs and holds none of the simulated method's arithmetic (no lane
map, no IDM, no lane change, no claims).  Routes are inputs to the method
("from the input demand data after the routing"); the router here is
a generator-side tool.

Configs (BASELINE.json ``configs``; recipes in DESIGN.md §5):
  grid4    C1  4x4 grid, 2 lanes, 100 m, 1,000 trips over 1 h
  grid4b   C1b same, departures in [0, 300) s (conflict stress)
  sfcity   C2  ~10k-node jittered city grid, ~100k trips over 3 h
  bay      C3  Bay-Area-shaped ~224k nodes / ~549k edges, 2.82M trips over 12 h
  bay9m    C4  same graph, 9,008,766 trips
  bay24m   C5  same graph, 24M trips over 24 h
"""
from .synth import (  # noqa: F401
    CONFIGS,
    grid_graph,
    make_workload,
    route_trips,
    graph_summary,
)
