"""CLI (paper_1604_06525_b200/cli.py; SPEC.md "cli" module, the reference's
tools/minopt_cli.cpp is a stub): usage / binding errors exit 2 without a GPU;
solves on the device reproduce the SPEC's examples (laplacian.opt: final
cost 1/3 at x = [2/3, 1/3]; --materialize jtj gives the same x within 1e-10;
compare's divergence column <= 1e-6; trace CSV with the reference's schema,
solver.hpp:66-74)."""
import os

import numpy as np
import pytest

from paper_1604_06525_b200 import cli
from paper_1604_06525_b200.optio import read_optd, write_optd

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LAP = os.path.join(ROOT, "examples", "laplacian", "laplacian.opt")
A = os.path.join(ROOT, "examples", "laplacian", "A.optd")


@pytest.mark.parametrize("argv,msg", [
    (["solve", LAP], "missing binding for A"),
    (["solve", LAP, "--bind", f"A={A}", "--bind", "Q=1"], "names nothing"),
    (["solve", LAP, "--bind", f"A={A}", "--bind", f"A={A}"], "bound twice"),
    (["solve", "/nonexistent.opt"], "not found"),
    (["solve", LAP, "--bind", "A=/nonexistent.optd"], "cannot open"),
    (["solve", LAP, "--bind", f"A={A}", "--dim", "Z=3"], "no declared dim"),
])
def test_usage_errors_exit_2(argv, msg, capsys):
    assert cli.main(argv) == 2
    assert msg in capsys.readouterr().err


def test_shape_mismatch_exit_2(tmp_path, capsys):
    bad = tmp_path / "A3.optd"
    write_optd(bad, np.zeros(3))
    assert cli.main(["solve", LAP, "--bind", f"A={bad}"]) == 2
    assert "holds 3 values" in capsys.readouterr().err


def test_compile_error_exit_2(tmp_path, capsys):
    p = tmp_path / "bad.opt"
    p.write_text("dim W 2\nunknown X [W]\nenergy X(0) +\n")
    assert cli.main(["solve", str(p)]) == 2
    assert "SyntaxError" in capsys.readouterr().err


@pytest.mark.gpu
def test_solve_laplacian(tmp_path, capsys):
    trace = tmp_path / "t.csv"
    rc = cli.main(["solve", LAP, "--bind", f"A={A}", "--method", "gn", "--nl-iters", "1", "--trace", str(trace),
                   "--out", str(tmp_path)])
    out = capsys.readouterr().out
    assert rc == 0
    cost = float(out.split("final_cost ")[1].split()[0])
    assert abs(cost - 1.0 / 3.0) <= 1e-12
    x = read_optd(tmp_path / "X.optd")
    assert x.extents == [2] and x.channels == 1
    np.testing.assert_allclose(x.values, [2 / 3, 1 / 3], rtol=0, atol=1e-12)
    lines = trace.read_text().splitlines()
    assert lines[0] == "iter,cost,accepted,radius,pcg_iters,wall_ms"
    assert lines[1].split(",")[:3] == ["0", repr(cost), "1"]
    rc = cli.main(["solve", LAP, "--bind", f"A={A}", "--nl-iters", "1", "--materialize", "jtj", "--out",
                   str(tmp_path / "jtj")])
    assert rc == 0
    np.testing.assert_allclose(read_optd(tmp_path / "jtj" / "X.optd").values, x.values, rtol=0, atol=1e-10)


@pytest.mark.gpu
def test_compare_modes(capsys):
    assert cli.main(["compare", LAP, "--bind", f"A={A}", "--nl-iters", "2"]) == 0
    rows = capsys.readouterr().out.strip().splitlines()
    assert rows[0] == "mode,ms_per_linear_iter,j_storage_bytes,max_rel_divergence,final_cost"
    modes = {r.split(",")[0]: r.split(",") for r in rows[1:]}
    assert set(modes) == {"matrix-free", "materialize=j", "materialize=jtj"}
    assert int(modes["matrix-free"][2]) == 0
    for m in modes.values():
        assert float(m[3]) <= 1e-6
