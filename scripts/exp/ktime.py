"""Unperturbed apply / build_normal time (mo_bench_kernel) of one config under
the current MO_B200_* environment:  python scripts/exp/ktime.py arap_warp 8192"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_1604_06525_b200 import Method, Precision, SolveConfig, Solver, load_plan, workloads
name = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
prob = {"arap_warp": lambda: workloads.arap_warp(n, n), "poisson": lambda: workloads.poisson(n, n),
        "sfs": lambda: workloads.sfs(640, 480), "arap_mesh": lambda: workloads.arap_mesh(448)}[name]()
cfg = SolveConfig(method=Method.kLevenbergMarquardt if prob.method == "lm" else Method.kGaussNewton,
                  precision=Precision.kF32, nonlinear_iters=1, linear_iters=2)
s = Solver(load_plan(prob.name, cfg, prob.dims), prob.data(np.float32))
s.solve()
a = min(s.bench_kernel(0, 20) for _ in range(2))
b = s.bench_kernel(1, 10)
env = {k[7:]: v for k, v in os.environ.items() if k.startswith("MO_B200_")}
print(json.dumps({"cfg": f"{name} {n}", "env": env, "apply": s.apply_kernel(0), "apply_us": round(a * 1e3, 1),
                  "normal": s.normal_kernel(0), "normal_us": round(b * 1e3, 1)}), flush=True)
