import os, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
from oracle import pyoracle
from paper_1604_06525_b200 import workloads, Solver, load_plan, Method, Precision, SolveConfig
prob = workloads.arap_mesh(448)
for prec in ("f32", "f64"):
    dt = np.float32 if prec == "f32" else np.float64
    cfg = SolveConfig(method=Method.kGaussNewton, precision=Precision.kF32 if prec == "f32" else Precision.kF64,
                      nonlinear_iters=2, linear_iters=20, pcg_rel_tol=0.0, pcg_abs_tol=0.0, cost_stop_tol=0.0)
    ref = pyoracle.run_ref(prob.energy, prob.data(dt), ["solve"], dims=prob.dims, prec=prec, nl=2, lin=20, rel=0.0,
                           abs_tol=0.0, cost_stop=0.0, exec_mode="par", threads=os.cpu_count())
    for fuse in ("1", None):
        if fuse: os.environ["MO_B200_NO_VFUSE"] = "1"
        else: os.environ.pop("MO_B200_NO_VFUSE", None)
        r = Solver(load_plan(prob.name, cfg, prob.dims), prob.data(dt)).solve()
        print(prec, "novfuse" if fuse else "vfuse", [t.cost for t in r.trace], "ref", list(ref["trace_cost"]), flush=True)
