"""Profile helper: linearize + a few applies of a materialized plan (for ncu)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import bench
from paper_1604_06525_b200 import Solver, load_plan

cfg_name, suffix = sys.argv[1], sys.argv[2]
prob = bench.make_problem(cfg_name, 0)
plan = load_plan(prob.name + suffix, bench.solve_config(prob, "f32"), prob.dims)
s = Solver(plan, prob.data(np.float32))
s.build_normal()
s.linearize()
v = np.ones(s.num_cols(), np.float32)
for _ in range(3):
    s.apply_jtj(v)
