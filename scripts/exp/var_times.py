"""Tuner timings (MO_B200_TUNE_LOG) of every J^T J p and build_normal kernel
on one config:  python scripts/exp/var_times.py arap_warp 8192"""
import os, sys
os.environ["MO_B200_TUNE_LOG"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_1604_06525_b200 import Method, Precision, SolveConfig, Solver, load_plan, workloads
name = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
prec = sys.argv[3] if len(sys.argv) > 3 else "f32"
prob = {"arap_warp": lambda: workloads.arap_warp(n, n), "poisson": lambda: workloads.poisson(n, n),
        "sfs": lambda: workloads.sfs(640, 480), "arap_mesh": lambda: workloads.arap_mesh(448)}[name]()
dt = np.float32 if prec == "f32" else np.float64
cfg = SolveConfig(method=Method.kLevenbergMarquardt if prob.method == "lm" else Method.kGaussNewton,
                  precision=Precision.kF32 if prec == "f32" else Precision.kF64, nonlinear_iters=1, linear_iters=2)
s = Solver(load_plan(prob.name, cfg, prob.dims), prob.data(dt))
print(name, n, prec, "apply", s.apply_kernel(0), "normal", s.normal_kernel(0), flush=True)
