"""Command-line front door (SPEC.md "cli" module; the reference ships only a
stub, tools/minopt_cli.cpp): compile an energy file with this package's own
front end, bind .optd / .optg data by name, solve on the device, write the
result arrays and the trace CSV.

    python -m paper_1604_06525_b200.cli solve PROBLEM.opt --bind NAME=FILE|VALUE ... \\
        [--dim NAME=N] [--method gn|lm] [--precision f32|f64] [--materialize none|j|jtj] \\
        [--nl-iters K] [--lin-iters L] [--pcg-rtol E] [--no-precond] [--seq|--par] \\
        [--trace out.csv] [--out DIR] [--device D]
    python -m paper_1604_06525_b200.cli compare PROBLEM.opt --bind ... [same flags]

Bindings: every declared array, graph and param must be bound exactly once
(arrays: .optd files, graphs: .optg files, params: literal numbers); an
unknown may be bound to an .optd file holding its initial value (default 0).
`solve` prints the termination reason and final cost, writes one
<unknown>.optd per unknown field into --out and the trace CSV
(iter,cost,accepted,radius,pcg_iters,wall_ms; SolveResult::trace_csv,
solver.hpp:66-74) to --trace.  `compare` runs the matrix-free, Materialize::kJ
and Materialize::kJtJ modes back to back and reports, per mode, the wall time
per linear iteration, the bytes of stored J (or H) and the largest relative
iterate divergence from the matrix-free run.

Exit codes (SPEC.md cli invariants): 0 success, 1 solver failure (non-finite
cost), 2 usage / compile / bind error.  --seq / --par select the reference's
CPU executor mode and are accepted for compatibility: the device executes
every pass in parallel, deterministically.
"""
import argparse
import os
import sys
import time

import numpy as np

from . import frontend
from ._lib import MoError
from .optio import read_optd, read_optg, write_optd
from .solver import CompiledPlan, Method, Precision, SolveConfig, SolveData, Solver, StopReason, to_string

USAGE_ERROR, SOLVER_FAILURE = 2, 1


class UsageError(Exception):
    pass


def _args(argv):
    ap = argparse.ArgumentParser(prog="mo_cli", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("solve", "compare"):
        p = sub.add_parser(name)
        p.add_argument("problem")
        p.add_argument("--bind", action="append", default=[], metavar="NAME=FILE|VALUE")
        p.add_argument("--dim", action="append", default=[], metavar="NAME=N")
        p.add_argument("--method", choices=["gn", "lm"], default="gn")
        p.add_argument("--precision", choices=["f32", "f64"], default="f64")
        p.add_argument("--materialize", choices=["none", "j", "jtj"], default="none")
        p.add_argument("--nl-iters", type=int, default=8)
        p.add_argument("--lin-iters", type=int, default=100)
        p.add_argument("--pcg-rtol", type=float, default=-1.0)
        p.add_argument("--no-precond", action="store_true")
        g = p.add_mutually_exclusive_group()
        g.add_argument("--seq", action="store_true")
        g.add_argument("--par", action="store_true")
        p.add_argument("--trace")
        p.add_argument("--out")
        p.add_argument("--device", type=int, default=0)
    sub.add_parser("nist").add_argument("suite_dir")
    return ap.parse_args(argv)


def _config(a):
    return SolveConfig(method=Method.kLevenbergMarquardt if a.method == "lm" else Method.kGaussNewton,
                       precision=Precision.kF32 if a.precision == "f32" else Precision.kF64,
                       nonlinear_iters=a.nl_iters, linear_iters=a.lin_iters, pcg_rel_tol=a.pcg_rtol,
                       use_preconditioner=not a.no_precond)


def _kv(items, what):
    out = {}
    for it in items:
        if "=" not in it:
            raise UsageError(f"{what} '{it}' is not NAME=VALUE")
        k, v = it.split("=", 1)
        if k in out:
            raise UsageError(f"'{k}' is bound twice")
        out[k] = v
    return out


def load_problem(a):
    """(spec, plan text, SolveData) of a command line; UsageError on any
    binding problem, MoError on compile errors."""
    if not os.path.exists(a.problem):
        raise UsageError(f"problem file '{a.problem}' not found")
    src = open(a.problem).read()
    dims = {k: int(v) for k, v in _kv(a.dim, "--dim").items()}
    spec = frontend.compile_source(src)
    if dims:
        unknown = set(dims) - {n for n, _ in spec.dims}
        if unknown:
            raise UsageError(f"--dim names no declared dim: {sorted(unknown)}")
        spec.dims = [(n, dims.get(n, e)) for n, e in spec.dims]
    binds = _kv(a.bind, "--bind")
    declared = ([u.name for u in spec.unknowns] + [x.name for x in spec.arrays] + [g for g, _ in spec.graphs] +
                list(spec.params))
    extra = set(binds) - set(declared)
    if extra:
        raise UsageError(f"--bind names nothing the problem declares: {sorted(extra)}")
    missing = [n for n in [x.name for x in spec.arrays] + [g for g, _ in spec.graphs] + list(spec.params)
               if n not in binds]
    if missing:
        raise UsageError(f"missing binding for {', '.join(missing)}")
    dt = np.float32 if a.precision == "f32" else np.float64

    def dense(name, fld):
        arr = read_optd(binds[name])
        n = spec.extent(fld.dom) * fld.channels
        if arr.value_count() != n or arr.channels != fld.channels:
            raise UsageError(f"'{name}': {binds[name]} holds {arr.value_count()} values in {arr.channels} channels, "
                             f"the problem needs {n} in {fld.channels}")
        return arr.values.astype(dt)

    xs = [dense(u.name, u) if u.name in binds else np.zeros(spec.extent(u.dom) * u.channels, dt)
          for u in spec.unknowns]
    arrays = [dense(x.name, x) for x in spec.arrays]
    graphs = []
    for g, slots in spec.graphs:
        e = read_optg(binds[g])
        if e.arity != len(slots):
            raise UsageError(f"'{g}': {binds[g]} has arity {e.arity}, the graph declares {len(slots)} slots")
        graphs.append(e)
    params = []
    for p in spec.params:
        try:
            params.append(float(binds[p]))
        except ValueError:
            raise UsageError(f"param '{p}' must be bound to a number, got '{binds[p]}'")
    data = SolveData(x=np.concatenate(xs) if xs else np.zeros(0, dt), arrays=arrays, params=params, graphs=graphs)
    return spec, src, data


def _plan(spec, cfg, materialize):
    return CompiledPlan(frontend.plan_text(spec, cfg, materialize=materialize), cfg)


def cmd_solve(a, out=None):
    out = out or sys.stdout
    spec, _, data = load_problem(a)
    cfg = _config(a)
    mat = {"none": 0, "j": 1, "jtj": 2}[a.materialize]
    s = Solver(_plan(spec, cfg, mat), data, device=a.device)
    r = s.solve()
    print(f"reason {to_string(r.reason)}", file=out)
    print(f"final_cost {r.final_cost!r}", file=out)
    if a.trace:
        with open(a.trace, "w") as f:
            f.write(r.trace_csv())
    if a.out:
        os.makedirs(a.out, exist_ok=True)
        col = 0
        for u in spec.unknowns:
            n = spec.extent(u.dom) * u.channels
            write_optd(os.path.join(a.out, u.name + ".optd"), data.x[col:col + n], channels=u.channels,
                       extents=spec.shape(u.dom))
            col += n
    return SOLVER_FAILURE if r.reason == StopReason.kNonFiniteCost or not np.isfinite(r.final_cost) else 0


def cmd_compare(a, out=None):
    out = out or sys.stdout
    spec, _, data0 = load_problem(a)
    cfg = _config(a)
    rows, x_free = [], None
    for label, mat in (("matrix-free", 0), ("materialize=j", 1), ("materialize=jtj", 2)):
        data = SolveData(x=np.array(data0.x), arrays=data0.arrays, params=data0.params, graphs=data0.graphs)
        s = Solver(_plan(spec, cfg, mat), data, device=a.device)
        s.solve()  # warm-up (module load, tuning, graph capture)
        data.x[:] = data0.x  # the timed solve starts from the same state
        s._bind_all()
        s.refresh()
        t0 = time.perf_counter()
        r = s.solve()
        wall = (time.perf_counter() - t0) * 1e3
        pcg = max(1, sum(t.pcg_iters for t in r.trace))
        jbytes = 0
        if mat:
            s.linearize()
            if mat == 1:
                offs, col, val = s.jacobian()
            else:
                offs, col, val = s.normal_matrix()
            jbytes = int(val.nbytes + col.nbytes + offs.nbytes)
        x = np.array(data.x, np.float64)
        if x_free is None:
            x_free = x
        div = float(np.max(np.abs(x - x_free)) / max(np.max(np.abs(x_free)), 1e-300)) if x.size else 0.0
        rows.append((label, wall / pcg, jbytes, div, r.final_cost))
    print("mode,ms_per_linear_iter,j_storage_bytes,max_rel_divergence,final_cost", file=out)
    for label, ms, jb, div, fc in rows:
        print(f"{label},{ms:.6g},{jb},{div:.3e},{fc!r}", file=out)
    return 0


def main(argv=None):
    a = _args(sys.argv[1:] if argv is None else argv)
    try:
        if a.cmd == "nist":
            print("nist: the NIST StRD problem files are not part of this environment (SPEC.md cli cmd_nist)",
                  file=sys.stderr)
            return USAGE_ERROR
        return cmd_solve(a) if a.cmd == "solve" else cmd_compare(a)
    except UsageError as e:
        print(f"error: {e}", file=sys.stderr)
        return USAGE_ERROR
    except MoError as e:
        print(f"error: {e}", file=sys.stderr)
        return SOLVER_FAILURE if e.code == "NonFiniteCost" else USAGE_ERROR


if __name__ == "__main__":
    sys.exit(main())
