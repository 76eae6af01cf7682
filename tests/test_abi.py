"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports
every symbol include/mo_b200.h declares, parses every shipped plan, and fails
loudly (NoDevice) instead of falling back to the CPU when no GPU is present."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_1604_06525_b200 import _lib, load_plan
from paper_1604_06525_b200.solver import PLAN_DIR

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "mo_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(mo_\w+)\(", text, re.M)))


def test_every_header_symbol_is_exported():
    syms = header_symbols()
    assert len(syms) >= 35
    for s in syms:
        assert hasattr(_lib.lib, s), s
        assert s in _lib.SIGNATURES, s


@pytest.mark.parametrize("name", ["poisson", "arap_warp", "arap_mesh", "sfs"])
def test_shipped_plans_parse(name):
    p = load_plan(name)
    assert p.num_cols > 0
    assert p.cfg.nonlinear_iters >= 1


def test_dim_override_recomputes_layout():
    p = load_plan("poisson", dims={"W": 16, "H": 12})
    assert p.num_cols == 16 * 12 * 3
    assert p.array_size(0) == 16 * 12 * 3 and p.array_size(1) == 16 * 12
    m = load_plan("arap_mesh", dims={"N": 64})
    assert m.num_cols == 64 * 6 and m.graph_arity(0) == 2


def test_bad_plan_text_is_a_format_error():
    with pytest.raises(_lib.MoError) as e:
        load_plan(os.path.join(PLAN_DIR, "poisson.moplan"))  # fine
        from paper_1604_06525_b200 import plan
        plan("moplan 1\ncfg 0 1")
    assert e.value.code in ("TruncatedFile", "FormatError")


def test_config_checks_follow_plan_hpp():
    from paper_1604_06525_b200 import SolveConfig
    with pytest.raises(_lib.MoError) as e:
        load_plan("poisson", SolveConfig(nonlinear_iters=0))
    assert e.value.code == "BindError"
    p = load_plan("poisson", SolveConfig(precision=0, pcg_rel_tol=-1))
    assert p.cfg.pcg_rel_tol == 1e-4  # plan.hpp:192-193


def test_no_cpu_fallback_without_gpu():
    from paper_1604_06525_b200 import SolveData, Solver, device_count
    if device_count() > 0:
        pytest.skip("GPU present")
    p = load_plan("poisson", dims={"W": 8, "H": 8})
    with pytest.raises(_lib.MoError) as e:
        Solver(p, SolveData(x=np.zeros(p.num_cols), arrays=[np.zeros(192), np.zeros(64)]))
    assert e.value.code == "NoDevice"


@pytest.mark.parametrize("name,mode", [("poisson", 0), ("poisson_mat", 1), ("arap_warp_math", 2), ("arap_mesh_mat", 1),
                                       ("arap_mesh_math", 2)])
def test_materialize_mode_travels_with_the_plan(name, mode):
    """Materialize (plan.hpp:17) is fixed at plan time: a kJ / kJtJ plan
    carries no gather J^T J programs (empty in the interchange) and keeps its
    mode across set_config."""
    from paper_1604_06525_b200 import SolveConfig
    p = load_plan(name)
    assert p.materialize == mode
    q = load_plan(name, SolveConfig(nonlinear_iters=3, linear_iters=5))
    assert q.materialize == mode
    text = open(os.path.join(PLAN_DIR, name + ".moplan")).read()
    assert ("program jtj 0 0 0 0 0" in text) == (mode != 0)


def test_workload_import_does_not_map_the_product_library():
    """bench.py's reference arm generates inputs with workloads.py; that must
    not dlopen libmo_b200.so (the library loads on first use only)."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_1604_06525_b200 import workloads\n"
            "workloads.poisson(8, 8)\n"
            "print(any('libmo_b200' in l for l in open('/proc/self/maps')))\n") % ROOT
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, check=True).stdout
    assert out.strip() == "False"


def test_pcg_operand_checks_precede_any_device_work():
    from paper_1604_06525_b200 import pcg
    b = np.ones(4)
    with pytest.raises(_lib.MoError):
        pcg(lambda x, y, s: None, b, np.ones(4), excluded=np.zeros(3, np.uint8))
    with pytest.raises(_lib.MoError):
        pcg(lambda x, y, s: None, b, np.ones(5))
