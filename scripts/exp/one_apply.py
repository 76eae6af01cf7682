"""A few build_normal + J^T J p launches of one config (for ncu -k captures):
    python scripts/exp/one_apply.py arap_warp|poisson|sfs|arap_mesh [size] [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_1604_06525_b200 import Method, Precision, SolveConfig, Solver, load_plan, workloads
name = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
prob = {"arap_warp": lambda: workloads.arap_warp(n, n), "poisson": lambda: workloads.poisson(n, n),
        "sfs": lambda: workloads.sfs(640, 480), "arap_mesh": lambda: workloads.arap_mesh(448)}[name]()
cfg = SolveConfig(method=Method.kLevenbergMarquardt if prob.method == "lm" else Method.kGaussNewton,
                  precision=Precision.kF32, nonlinear_iters=1, linear_iters=2)
s = Solver(load_plan(prob.name, cfg, prob.dims), prob.data(np.float32))
v = (workloads.uniform(97, s.num_cols()) - 0.5).astype(np.float32)
for _ in range(reps):
    s.build_normal()
    s.apply_jtj(v)
print("apply", s.apply_kernel(0), "normal", s.normal_kernel(0))
