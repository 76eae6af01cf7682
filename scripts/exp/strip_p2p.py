"""Time LocalComm strip solves with / without peer reductions:
    python scripts/exp/strip_p2p.py arap_warp 2048 4"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_1604_06525_b200 import Method, Precision, SolveConfig, load_plan, workloads
from paper_1604_06525_b200.sharded import LocalShardGroup
name, n, world = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
prob = workloads.poisson(n, n) if name == "poisson" else workloads.arap_warp(n, n)
cfg = SolveConfig(method=Method.kGaussNewton, precision=Precision.kF32, nonlinear_iters=1, linear_iters=10,
                  pcg_rel_tol=0.0)
for rep in range(2):
    g = LocalShardGroup(load_plan(prob.name, cfg, prob.dims), prob.data(np.float32), world)
    t0 = time.time()
    try:
        res = g.solve()
        print(name, n, world, "p2p" if not os.environ.get("MO_B200_NO_P2P") else "nccl-path", rep,
              round(time.time() - t0, 2), "s", res[0].final_cost, flush=True)
    except Exception as e:
        print("ERROR", rep, round(time.time() - t0, 2), e, flush=True)
    finally:
        g.close()
