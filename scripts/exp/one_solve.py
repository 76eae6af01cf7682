"""One GN iteration (20 PCG) of a config, for ncu launch lists:
    python scripts/exp/one_solve.py arap_warp 8192 [nl]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_1604_06525_b200 import Method, Precision, SolveConfig, Solver, load_plan, workloads
name = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
nl = int(sys.argv[3]) if len(sys.argv) > 3 else 1
prob = {"arap_warp": lambda: workloads.arap_warp(n, n), "poisson": lambda: workloads.poisson(n, n),
        "sfs": lambda: workloads.sfs(640, 480), "arap_mesh": lambda: workloads.arap_mesh(448)}[name]()
cfg = SolveConfig(method=Method.kLevenbergMarquardt if prob.method == "lm" else Method.kGaussNewton,
                  precision=Precision.kF32, nonlinear_iters=nl, linear_iters=20, pcg_rel_tol=0.0, pcg_abs_tol=0.0,
                  cost_stop_tol=0.0)
s = Solver(load_plan(prob.name, cfg, prob.dims), prob.data(np.float32))
s.solve()
print("MARK", flush=True)
l0 = s.kernel_launches()
r = s.solve()
print("LAUNCHES", s.kernel_launches() - l0)
print(name, n, "final", r.final_cost, "apply", s.apply_kernel(0), "normal", s.normal_kernel(0))
