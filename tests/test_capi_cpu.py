"""CPU-side checks of the product boundary: the C-ABI library builds, loads and
exports every symbol include/lpsim.h declares; the struct layouts of the
binding match the header; without a GPU it fails loudly (no CPU fallback)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from tests.conftest import ROOT, cuda_available


def header_functions():
    src = open(os.path.join(ROOT, "include", "lpsim.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lpsim_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def built():
    from paper_2406_08496_b200 import build

    build.build()
    import paper_2406_08496_b200 as pkg

    return pkg.lib()


def test_library_exports_every_header_symbol(built):
    names = header_functions()
    assert "lpsim_create" in names and "lpsim_step" in names and "lpsim_results" in names
    for n in names:
        assert hasattr(built, n), n


def test_binding_exports_match_header():
    from paper_2406_08496_b200 import lpsim

    assert sorted(lpsim.EXPORTED) == header_functions()


def test_struct_sizes_match_header(built, tmp_path):
    """Compile a tiny C program against include/lpsim.h and compare sizeof."""
    from paper_2406_08496_b200.lpsim import Config, Graph, Stats

    prog = tmp_path / "s.c"
    prog.write_text('#include "lpsim.h"\n#include <stdio.h>\n#include <stddef.h>\n'
                    'int main(void){printf("%zu %zu %zu %zu %zu\\n", sizeof(lpsim_graph), sizeof(lpsim_config),'
                    ' sizeof(lpsim_stats), offsetof(lpsim_config, seed), offsetof(lpsim_config, flags));return 0;}\n')
    exe = tmp_path / "s"
    import subprocess

    subprocess.check_call(["gcc", "-I" + os.path.join(ROOT, "include"), str(prog), "-o", str(exe)])
    out = subprocess.check_output([str(exe)]).decode().split()
    assert int(out[0]) == C.sizeof(Graph)
    assert int(out[1]) == C.sizeof(Config)
    assert int(out[2]) == C.sizeof(Stats)
    assert int(out[3]) == Config.seed.offset
    assert int(out[4]) == Config.flags.offset


def test_config_defaults(built):
    from paper_2406_08496_b200 import default_config

    c = default_config()
    assert c.dt_s == 0.5 and c.a == 1.5 and c.delta == 4 and c.num_parts == 1 and c.seed == 1


@pytest.mark.skipif(cuda_available(), reason="checks the no-GPU failure path")
def test_no_gpu_fails_loudly(built):
    from paper_2406_08496_b200 import LpsimError, Simulation
    from tests.helpers import graph_from_edges

    g = graph_from_edges(2, [(0, 1, 100.0, 1, 13.9), (1, 0, 100.0, 1, 13.9)])
    with pytest.raises(LpsimError) as ei:
        Simulation(g)
    assert ei.value.status == 7  # LPSIM_E_CUDA


def test_validation_runs_before_device(built):
    """Graph validation errors are reported (with the offending index) even without a GPU."""
    from paper_2406_08496_b200 import LpsimError, Simulation
    from tests.helpers import graph_from_edges

    g = graph_from_edges(2, [(0, 1, 100.0, 1, 13.9), (1, 0, 100.0, 0, 13.9)])
    with pytest.raises(LpsimError) as ei:
        Simulation(g)
    assert ei.value.status == 2 and "index 1" in str(ei.value)
    g = graph_from_edges(2, [(0, 1, 100.0, 1, 13.9), (1, 0, 100.0, 1, 300.0)])
    with pytest.raises(LpsimError) as ei:
        Simulation(g)
    assert ei.value.status == 2

