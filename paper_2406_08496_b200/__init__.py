"""B200-native LPSim per-timestep vehicle update (arXiv 2406.08496).

The product is the C-ABI library ``liblpsim.so`` (include/lpsim.h) built from
``csrc/``; :mod:`.lpsim` is its thin Python binding.
"""
from .lpsim import (  # noqa: F401
    FLAG_CHECKS,
    FLAG_DIGESTS,
    FLAG_EDGE_TIMES,
    FLAG_NO_SORT,
    FLAG_RACY,
    FLAG_VFREE,
    FLAG_TIMING,
    LpsimError,
    Simulation,
    default_config,
    lib,
)
