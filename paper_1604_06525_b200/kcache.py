"""Ahead-of-time NVRTC compilation of the shipped plans into the in-tree kernel
cache (paper_1604_06525_b200/_kcache), so a fresh GPU box loads cubins instead
of compiling at session creation."""
import os

from ._lib import call
from .solver import PLAN_DIR, load_plan


def precompile_shipped():
    for f in sorted(os.listdir(PLAN_DIR)):
        if f.endswith(".moplan"):
            p = load_plan(os.path.join(PLAN_DIR, f))
            for prec in (0, 1):
                call("mo_plan_precompile", p._h, prec)
