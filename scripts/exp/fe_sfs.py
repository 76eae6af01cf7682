import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, "tests"); sys.path.insert(0, "tests/golden")
import numpy as np
from helpers import Golden
from paper_1604_06525_b200 import frontend, Solver
from paper_1604_06525_b200.solver import CompiledPlan
import test_frontend as tf
name = sys.argv[1] if len(sys.argv) > 1 else "cfg_sfs_f64"
g = Golden(name)
src, dims, mat = tf._source(name)
text = frontend.plan_source(src, g.cfg, dims=dims, materialize=mat)
s = Solver(CompiledPlan(text, g.cfg), g.data())
for step in sys.argv[2:] or ["cost", "normal", "jtj", "solve"]:
    print(step, flush=True)
    if step == "cost": print(s.cost())
    if step == "normal": s.build_normal()
    if step == "jtj": s.apply_jtj(g.z["v"].astype(g.dtype))
    if step == "solve": print(s.solve().final_cost)
