"""Ahead-of-time NVRTC compilation of the shipped plans into the in-tree kernel
cache (paper_1604_06525_b200/_kcache), so a fresh GPU box loads cubins instead
of compiling at session creation."""
import os

from ._lib import call
from .solver import PLAN_DIR, load_plan


# Grid sizes other than a plan's own that the benchmark and the full-size
# tests run (the plan's dims are compile-time constants of its kernels).
EXTRA_DIMS = {"arap_warp": [{"W": 8192, "H": 8192}, {"W": 2048, "H": 2048}],
              "poisson": [{"W": 8192, "H": 8192}, {"W": 2048, "H": 2048}]}


def precompile_shipped():
    for f in sorted(os.listdir(PLAN_DIR)):
        if f.endswith(".moplan"):
            p = load_plan(os.path.join(PLAN_DIR, f))
            for prec in (0, 1):
                call("mo_plan_precompile", p._h, prec)
            for dims in EXTRA_DIMS.get(f[:-7], []):
                q = load_plan(os.path.join(PLAN_DIR, f), dims=dims)
                call("mo_plan_precompile", q._h, 0)
