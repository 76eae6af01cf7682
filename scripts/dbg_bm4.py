import os, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
from paper_1604_06525_b200 import workloads, Solver, load_plan, Method, Precision, SolveConfig
from oracle import pyoracle
prob = workloads.arap_warp(1024, 1024)
cfg = SolveConfig(method=Method.kGaussNewton, precision=Precision.kF32, nonlinear_iters=10, linear_iters=20,
                  pcg_rel_tol=0.0, pcg_abs_tol=0.0, cost_stop_tol=0.0)
out = {}
for v in ("0", "1"):
    if v == "1": os.environ["MO_B200_NO_BM4"] = "1"
    else: os.environ.pop("MO_B200_NO_BM4", None)
    s = Solver(load_plan(prob.name, cfg, prob.dims), prob.data(np.float32))
    s.build_normal()
    out[v] = (np.array(s.rhs(), np.float64), np.array(s.precond(), np.float64))
    r = s.solve()
    print("nobm4", v, [round(t.cost, 5) for t in r.trace], flush=True)
for k, name in ((0, "b"), (1, "m")):
    a, b = out["0"][k], out["1"][k]
    d = np.abs(a - b); rel = d / np.maximum(np.abs(b), 1e-30)
    i = int(np.argmax(rel * (np.abs(b) > 1e-6 * np.abs(b).max())))
    print(name, "max abs", d.max(), "scale", np.abs(b).max(), "worst rel (non-tiny)", rel[i], a[i], b[i], i)
ref = pyoracle.run_ref(prob.energy, prob.data(np.float64), ["solve", "normal"], dims=prob.dims, prec="f64", nl=10, lin=20, rel=0.0,
                       abs_tol=0.0, cost_stop=0.0, exec_mode="par", threads=os.cpu_count())
print("ref f64", [round(c, 5) for c in ref["trace_cost"]])
for k, name in ((0, "b"), (1, "m")):
    rr = ref[name]
    for v in ("0", "1"):
        a = out[v][k]; d = np.abs(a - rr); rel = d / np.maximum(np.abs(rr), 1e-30)
        big = np.abs(rr) > 1e-6 * np.abs(rr).max()
        print(name, "nobm4", v, "max rel (non-tiny) vs f64 ref", rel[big].max(), "count>1e-5", int((rel[big] > 1e-5).sum()))
