"""Regenerate the golden fixtures from the UNMODIFIED reference.

    make -C oracle && make -C integration && python tests/golden/make_golden.py

Needs /root/reference (this container only).  Writes, per case:
  <name>.moplan   plan exported by integration/_build/export_plan
  <name>.npz      inputs + cfg + reference outputs (keys ref_*)
"""
import json
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from cases import CONFIG_CASES, unit_cases  # noqa: E402
from oracle import pyoracle  # noqa: E402
from paper_1604_06525_b200 import workloads  # noqa: E402
from paper_1604_06525_b200.solver import EdgeTable, SolveData  # noqa: E402

EXPORT = os.path.join(ROOT, "integration", "_build", "export_plan")


def export(src_or_path, dims=None, cfg=None):
    with tempfile.TemporaryDirectory() as td:
        path = pyoracle.energy_path(src_or_path, td)
        cmd = [EXPORT, "--energy", path]
        if (cfg or {}).get("materialize"):
            cmd += ["--materialize", cfg["materialize"]]
        for k, v in (dims or {}).items():
            cmd += ["--dim", f"{k}={v}"]
        return subprocess.run(cmd, check=True, capture_output=True, text=True).stdout


def run_case(name, src, data, cfg, prec, cmds, v, dims=None, energy=None):
    plan_text = export(energy or src, dims, cfg)
    with open(os.path.join(HERE, name + ".moplan"), "w") as f:
        f.write(plan_text)
    kw = dict(prec=prec, method=cfg.get("method", "gn"), nl=cfg.get("nl"), lin=cfg.get("lin"),
              rel=cfg.get("rel"), radius0=cfg.get("radius0"), cost_stop=cfg.get("cost_stop"), v=v, dims=dims,
              materialize=cfg.get("materialize"), force_evalj=cfg.get("force_evalj", False))
    out = pyoracle.run_ref(energy or src, data, cmds, **kw)
    rec = {"x": np.asarray(data.x, np.float64), "params": np.asarray(data.params, np.float64),
           "prec": np.array(prec), "cfg": np.array(json.dumps(cfg)), "cmds": np.array(",".join(cmds)),
           "n_arrays": np.array(len(data.arrays)), "n_graphs": np.array(len(data.graphs))}
    for i, a in enumerate(data.arrays):
        rec[f"array{i}"] = np.asarray(a, np.float64)
    for i, g in enumerate(data.graphs):
        rec[f"graph{i}"] = np.asarray(g.verts, np.uint64)
        rec[f"graph{i}_arity"] = np.array(g.arity)
    if v is not None:
        rec["v"] = np.asarray(v, np.float64)
    for k, val in out.items():
        rec["ref_" + k] = val
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **rec)
    err = out.get("error")
    print(f"{name:20s} {'ERROR ' + bytes(err).decode() if err is not None else 'ok'}")


def main():
    only = set(sys.argv[1:])  # optional: regenerate just these case names
    for name, c in unit_cases().items():
        if only and name not in only:
            continue
        dt = np.float32 if c["prec"] == "f32" else np.float64
        data = SolveData(x=np.asarray(c["x"], dt), arrays=[np.asarray(a, dt) for a in c["arrays"]],
                         params=c["params"], graphs=[EdgeTable(a, np.asarray(v, np.uint64)) for a, v in c["graphs"]])
        run_case(name, c["src"], data, c["cfg"], c["prec"], c["cmds"], c["v"])
    for name, (wl, kw, cfg) in CONFIG_CASES.items():
        prob = workloads.CONFIGS[wl](**kw)
        for prec in ("f64", "f32"):
            if only and f"{name}_{prec}" not in only:
                continue
            dt = np.float32 if prec == "f32" else np.float64
            data = prob.data(dt)
            v = workloads.uniform(99, data.x.size) - 0.5
            cmds = ["cost", "residuals", "normal", "jtj", "solve"]
            if cfg.get("materialize"):
                cmds = ["cost", "residuals", "normal", "linearize", "jtj", "solve"]
            run_case(f"{name}_{prec}", None, data, cfg, prec, cmds, v.astype(dt), dims=prob.dims, energy=prob.energy)


if __name__ == "__main__":
    main()
