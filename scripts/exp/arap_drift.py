"""ARAP 1024^2 fp32 10x20 trajectory under forced build_normal / apply kernels
vs the fp64 reference trajectory (measured on this host's reference)."""
import os, sys, subprocess, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
REF64 = [1901.6960792062428, 1580.5443358208513, 1466.4791582171324, 1397.3790015120571, 1345.9108832692484,
         1305.383068104849, 1271.3169845155358, 1242.2874052562408, 1216.08324742313, 1192.9803100328352]
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import numpy as np
    from paper_1604_06525_b200 import Method, Precision, SolveConfig, Solver, load_plan, workloads
    prob = workloads.arap_warp(1024, 1024)
    cfg = SolveConfig(method=Method.kGaussNewton, precision=Precision.kF32, nonlinear_iters=10, linear_iters=20,
                      pcg_rel_tol=0.0, pcg_abs_tol=0.0, cost_stop_tol=0.0)
    s = Solver(load_plan(prob.name, cfg, prob.dims), prob.data(np.float32))
    r = s.solve()
    errs = [abs(t.cost - c) / c for t, c in zip(r.trace, REF64)]
    print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("MO_B200")},
                      "apply": s.apply_kernel(0), "bm": s.normal_kernel(0), "final": r.final_cost,
                      "max_rel": max(errs), "rels": ["%.1e" % e for e in errs]}), flush=True)
    sys.exit(0)
for bm in ("prog", "bm4"):
    for jtj in ("tma", "gather", "tma4", "warp"):
        env = dict(os.environ, MO_B200_BM=bm, MO_B200_JTJ=jtj)
        subprocess.run([sys.executable, __file__, "child"], env=env)
