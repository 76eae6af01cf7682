"""Reference CPU rows of SURVEY §8d: the unmodified minopt on this host, one
GN/LM iteration of each config, fp32 and fp64, all host threads and 1 thread
(median of `--repeat` IterRow.wall_ms).  One JSON line per row."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from oracle import pyoracle  # noqa: E402

repeat = int(sys.argv[1]) if len(sys.argv) > 1 else 2
for cfg in ("arap_warp", "poisson", "arap_mesh"):
    prob = bench.make_problem(cfg, 0)
    for prec in ("f32", "f64"):
        for threads in (os.cpu_count(), 1):
            data = prob.data(np.float32 if prec == "f32" else np.float64)
            out = pyoracle.run_ref(prob.energy, data, ["time"], dims=prob.dims, prec=prec, method=prob.method, nl=1,
                                   lin=bench.LIN, rel=0.0, abs_tol=0.0, cost_stop=0.0, exec_mode="par",
                                   repeat=repeat, threads=threads)
            print(json.dumps({"config": bench.workload_name(prob), "prec": prec, "threads": threads,
                              "reference_ms_per_iter": float(np.median(out["time_row_ms"]))}), flush=True)
