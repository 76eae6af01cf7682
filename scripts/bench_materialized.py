"""Materialize modes on B200 vs the reference's CPU (
the paper's Figs. 16/17 trade-off between matrix-free and materialized J).

For each config and mode (matrix-free, Materialize::kJ, Materialize::kJtJ):
  * device: ms per GN iteration of solve() (10 nl x 20 PCG, fixed iterations,
    inputs resident, CUDA events on the session stream), plus the average
    apply and linearize times from the session's profiling hooks;
  * reference: the unmodified minopt (oracle/_ref/ref_driver) in the same
    mode on all host threads, one GN iteration per repeat (IterRow.wall_ms).
Prints one JSON line per (config, mode).

    python scripts/bench_materialized.py [--configs poisson,arap_warp,arap_mesh] [--ref-repeat 2]
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1604_06525_b200 import Solver, load_plan  # noqa: E402
from paper_1604_06525_b200 import _lib  # noqa: E402
from paper_1604_06525_b200._lib import call  # noqa: E402

MODES = {"free": ("", None), "kJ": ("_mat", "j"), "kJtJ": ("_math", "jtj")}


def device_ms(prob, suffix, prec, steps, warmup):
    cfg = bench.solve_config(prob, prec)
    plan = load_plan(prob.name + suffix, cfg, prob.dims)
    data = prob.data(np.float32 if prec == "f32" else np.float64)
    s = Solver(plan, data)
    stream = ctypes.c_void_p()
    call("mo_session_stream", s._h, ctypes.byref(stream))
    st = torch.cuda.ExternalStream(stream.value)
    res = _lib.SolveResultC()
    null_cb = _lib.ITER_CB()

    x0 = np.ascontiguousarray(data.x)

    def solve():  # rebind the start point (on the stream, before the timed solve)
        call("mo_bind_x", s._h, x0.ctypes.data, x0.size)
        call("mo_solve", s._h, null_cb, None, ctypes.byref(res))

    for _ in range(warmup):
        solve()
    times = []
    for _ in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        call("mo_bind_x", s._h, x0.ctypes.data, x0.size)
        torch.cuda.synchronize()
        a.record(st)
        call("mo_solve", s._h, null_cb, None, ctypes.byref(res))
        b.record(st)
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b) / bench.NL)
    call("mo_set_profiling", s._h, 1)
    solve()
    ms, n = ctypes.c_double(), ctypes.c_int64()
    call("mo_profile_read", s._h, 0, ctypes.byref(ms), ctypes.byref(n))
    apply_us = ms.value / max(n.value, 1) * 1e3
    return float(np.median(times)), apply_us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="poisson,arap_warp,arap_mesh")
    ap.add_argument("--prec", default="f32")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--ref-repeat", type=int, default=2)
    args = ap.parse_args()
    from oracle import pyoracle
    for cname in args.configs.split(","):
        prob = bench.make_problem(cname, 0)
        for mode, (suffix, mat) in MODES.items():
            line = {"config": bench.workload_name(prob), "mode": mode, "prec": args.prec}
            try:
                line["device_ms_per_iter"], line["device_apply_us"] = device_ms(prob, suffix, args.prec, args.steps,
                                                                                 args.warmup)
            except Exception as e:  # noqa: BLE001
                line["device_error"] = str(e)
            if args.ref_repeat > 0 and pyoracle.ref_available():
                data = prob.data(np.float32 if args.prec == "f32" else np.float64)
                out = pyoracle.run_ref(prob.energy, data, ["time"], dims=prob.dims, prec=args.prec,
                                       method=prob.method, nl=1, lin=bench.LIN, rel=0.0, abs_tol=0.0, cost_stop=0.0,
                                       exec_mode="par", repeat=args.ref_repeat, threads=os.cpu_count(),
                                       materialize=mat)
                line["reference_ms_per_iter"] = float(np.median(out["time_row_ms"]))
                line["reference_threads"] = os.cpu_count()
            print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
