"""Own front end (paper_1604_06525_b200/frontend.py) against the UNMODIFIED
reference, on the CPU (no GPU needed):

* every golden case (the reference's unit tests and the four BASELINE
  energies, tests/golden) is re-planned from its energy text by the front
  end and executed by the C restatement of run_program / exec / the solver
  (oracle/, the checker) on the golden's inputs: cost, residuals, b, m,
  2 J^T J v and the whole solve trajectory must equal the reference's outputs
  to rounding (the programs are the front end's own, not the reference's
  instruction streams);
* malformed sources fail with the Err the reference raises for them
  (tests/golden/frontend/errors.json, make_frontend_golden.py);
* the accepted "ok_*" sources plan and evaluate like the reference (live
  oracle/_ref/ref_driver on seeded data).
"""
import json
import os
import sys

import numpy as np
import pytest

from helpers import GOLDEN, Golden, golden_names
from oracle import pyoracle
from oracle.cref import Oracle
from paper_1604_06525_b200 import MoError, frontend, workloads
from paper_1604_06525_b200.solver import SolveConfig, SolveData

sys.path.insert(0, GOLDEN)
import cases  # noqa: E402

MAT = {None: 0, "j": 1, "jtj": 2}
UNIT = cases.unit_cases()
ERRORS = json.load(open(os.path.join(GOLDEN, "frontend", "errors.json")))


def _source(name):
    """(energy text, dims, materialize) of a golden case."""
    if name in UNIT:
        c = UNIT[name]
        return c["src"], None, MAT[c.get("cfg", {}).get("materialize")]
    for cname in sorted(cases.CONFIG_CASES, key=len, reverse=True):  # longest prefix (cfg_x_mat before cfg_x)
        if name in (cname + "_f32", cname + "_f64"):
            wl, kw, cfg = cases.CONFIG_CASES[cname]
            prob = workloads.CONFIGS[wl](**kw)
            return open(pyoracle.energy_path(prob.energy)).read(), prob.dims, MAT[cfg.get("materialize")]
    return None


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    if a.size == 0:
        return 0.0
    same = (a == b) | (np.isnan(a) & np.isnan(b))
    if same.all():
        return 0.0
    return float(np.max(np.abs(a - b)[~same]) / max(float(np.max(np.abs(b[np.isfinite(b)]), initial=0.0)), 1e-300))


CASES = [n for n in golden_names() if _source(n) is not None]


@pytest.mark.parametrize("name", CASES)
def test_frontend_plan_matches_reference(name):
    g = Golden(name)
    if g.ref("error") is not None:
        pytest.skip("the reference raised for this case (checked on the device by test_golden_gpu)")
    src, dims, mat = _source(name)
    text = frontend.plan_source(src, g.cfg, dims=dims, materialize=mat)
    o = Oracle(text, f64=g.prec == "f64", cfg=g.cfg)
    o.bind(g.data())
    f64 = g.prec == "f64"
    vec, traj = (1e-12, 1e-9) if f64 else (2e-5, 1e-4)
    assert o.num_cols() == int(g.ref("num_cols")[0]) and o.num_rows() == int(g.ref("num_rows")[0])
    np.testing.assert_array_equal(o.excluded(), g.ref("excluded"))
    for cmd in g.cmds:
        if cmd == "cost":
            assert _rel([o.cost()], g.ref("cost")) <= vec
        elif cmd == "residuals":
            assert _rel(o.residuals(), g.ref("residuals")) <= vec * 10
        elif cmd == "normal":
            b, m = o.build_normal()
            assert _rel(b, g.ref("b")) <= vec * 10, "b"
            assert _rel(m, g.ref("m")) <= vec * 10, "m"
        elif cmd == "linearize":
            o.linearize()
        elif cmd == "jtj":
            assert _rel(o.apply_jtj(g.z["v"].astype(g.dtype)), g.ref("jtj")) <= vec * 10, "2 J^T J v"
        elif cmd == "solve":
            r, tr = o.solve()
            assert int(r.reason) == int(g.ref("reason")[0])
            assert list(tr["pcg"]) == list(g.ref("trace_pcg"))
            assert list(tr["accepted"]) == list(g.ref("trace_accepted"))
            for c, rc in zip(tr["cost"], g.ref("trace_cost")):
                assert _rel([c], [rc]) <= traj, (c, rc)
            assert _rel([r.final_cost], g.ref("final_cost")) <= traj


@pytest.mark.parametrize("name", sorted(ERRORS))
def test_frontend_errors_like_reference(name):
    case = ERRORS[name]
    if case["reference"] == "ok":
        frontend.plan_source(case["source"])
        return
    with pytest.raises(MoError) as ei:
        frontend.plan_source(case["source"])
    assert ei.value.code == case["reference"], str(ei.value)


@pytest.mark.skipif(not pyoracle.ref_available(), reason="oracle/_ref/ref_driver not built")
@pytest.mark.parametrize("name", [n for n in sorted(ERRORS) if ERRORS[n]["reference"] == "ok"])
def test_frontend_accepted_sources_evaluate_like_reference(name):
    src = ERRORS[name]["source"]
    spec = frontend.compile_source(src)
    rng = np.random.default_rng(7)
    ncols = sum(spec.extent(u.dom) * u.channels for u in spec.unknowns)
    data = SolveData(x=rng.uniform(0.2, 1.0, ncols),
                     arrays=[rng.uniform(0.1, 0.9, spec.extent(a.dom) * a.channels) for a in spec.arrays],
                     params=list(rng.uniform(0.5, 1.5, len(spec.params))), graphs=[])
    if spec.graphs:
        pytest.skip("no graph data in this case")
    v = rng.uniform(-1, 1, ncols)
    ref = pyoracle.run_ref(src, data, ["cost", "normal", "jtj"], v=v)
    cfg = SolveConfig()
    o = Oracle(frontend.plan_source(src, cfg), f64=True, cfg=cfg)
    o.bind(data)
    assert _rel([o.cost()], ref["cost"]) <= 1e-12
    b, m = o.build_normal()
    assert _rel(b, ref["b"]) <= 1e-11 and _rel(m, ref["m"]) <= 1e-11
    assert _rel(o.apply_jtj(v), ref["jtj"]) <= 1e-11


def test_plan_api_accepts_sources_and_paths(tmp_path):
    """plan() takes moplan text, energy text or a .opt path (front end);
    dims override declared extents."""
    from paper_1604_06525_b200 import plan
    src = "dim W 8\nunknown X [W]\narray A [W]\nenergy X(0) - A(0)\nenergy X(0) - X(1)\n"
    p = tmp_path / "chain.opt"
    p.write_text(src)
    for s in (src, str(p)):
        pl = plan(s, dims={"W": 16})
        assert pl.num_cols == 16
    text = frontend.plan_source(src)
    assert plan(text).num_cols == 8
