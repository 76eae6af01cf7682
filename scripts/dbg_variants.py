import os, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
from paper_1604_06525_b200 import workloads, Solver, load_plan, Method, Precision, SolveConfig
prob = workloads.arap_warp(1024, 1024)
cfg = SolveConfig(method=Method.kGaussNewton, precision=Precision.kF32, nonlinear_iters=2, linear_iters=10,
                  pcg_rel_tol=0.0, pcg_abs_tol=0.0, cost_stop_tol=0.0)
for v in sys.argv[1:]:
    os.environ['MO_B200_JTJ'] = v
    s = Solver(load_plan(prob.name, cfg, prob.dims), prob.data(np.float32))
    k = s.apply_kernel(0)
    r = s.solve()
    print(v, k, [round(t.cost, 4) for t in r.trace], r.final_cost, flush=True)
