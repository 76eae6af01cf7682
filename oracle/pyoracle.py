"""Python side of the oracle (TEST INFRASTRUCTURE ONLY).

* mob_write / mob_read: the tagged-blob container of oracle/mob.h.
* run_ref(...): run the UNMODIFIED reference solver (oracle/_ref/ref_driver,
  built from /root/reference headers by oracle/Makefile) on given inputs.
* C restatement (oracle/mo_oracle.c) bindings live in oracle/cref.py.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
arm may import this module.
"""
import os
import struct
import subprocess
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DRIVER = os.path.join(HERE, "_ref", "ref_driver")
ENERGY_DIR = os.path.join(os.path.dirname(HERE), "paper_1604_06525_b200", "energies")

_DT = {0: np.float32, 1: np.float64, 2: np.uint8, 3: np.int32, 4: np.int64, 5: np.uint64}
_CODE = {np.dtype(v): k for k, v in _DT.items()}


def mob_write(path, recs):
    with open(path, "wb") as f:
        f.write(b"MOB1")
        f.write(struct.pack("<I", len(recs)))
        for name, arr in recs.items():
            arr = np.ascontiguousarray(arr)
            nb = name.encode()
            f.write(struct.pack("<H", len(nb)))
            f.write(nb)
            f.write(struct.pack("<BQ", _CODE[arr.dtype], arr.size))
            f.write(arr.tobytes())


def mob_read(path):
    out = {}
    with open(path, "rb") as f:
        assert f.read(4) == b"MOB1"
        (n,) = struct.unpack("<I", f.read(4))
        for _ in range(n):
            (ln,) = struct.unpack("<H", f.read(2))
            name = f.read(ln).decode()
            dt, cnt = struct.unpack("<BQ", f.read(9))
            dtype = np.dtype(_DT[dt])
            out[name] = np.frombuffer(f.read(cnt * dtype.itemsize), dtype=dtype).copy()
    return out


def ref_available():
    return os.path.exists(REF_DRIVER)


def energy_path(stem_or_path, tmpdir=None):
    """Energy file for a stem, a path, or inline source text (written to tmpdir)."""
    if "\n" in stem_or_path or "energy " in stem_or_path or stem_or_path.startswith("dim "):
        p = os.path.join(tmpdir or tempfile.mkdtemp(), "energy.opt")
        with open(p, "w") as f:
            f.write(stem_or_path)
        return p
    if os.path.exists(stem_or_path):
        return stem_or_path
    return os.path.join(ENERGY_DIR, stem_or_path + ".opt")


def run_ref(energy, data, cmds, dims=None, prec="f64", method="gn", nl=None, lin=None, rel=None,
            abs_tol=None, precond=True, radius0=None, cost_stop=None, exec_mode="seq", repeat=1,
            v=None, threads=None, timeout=3600, materialize=None, force_evalj=False):
    """Run the reference solver; `data` is a SolveData-like object (x, arrays,
    params, graphs).  Returns the output record dict (see ref_driver.cpp)."""
    if not ref_available():
        raise RuntimeError(f"{REF_DRIVER} not built (make -C oracle)")
    with tempfile.TemporaryDirectory() as td:
        fin, fout = os.path.join(td, "in.mob"), os.path.join(td, "out.mob")
        dt = np.float32 if prec == "f32" else np.float64
        recs = {"x": np.asarray(data.x, dt)}
        for i, a in enumerate(data.arrays):
            recs[f"array{i}"] = np.asarray(a, dt)
        recs["params"] = np.asarray(data.params, np.float64)
        for i, g in enumerate(data.graphs):
            recs[f"graph{i}"] = np.asarray(g.verts, np.uint64)
            recs[f"graph{i}_arity"] = np.asarray([g.arity], np.int64)
        if v is not None:
            recs["v"] = np.asarray(v, dt)
        mob_write(fin, recs)
        cmd = [REF_DRIVER, "--energy", energy_path(energy, td), "--in", fin, "--out", fout,
               "--prec", prec, "--method", method, "--exec", exec_mode, "--repeat", str(repeat),
               "--do", ",".join(cmds)]
        for k, val in (dims or {}).items():
            cmd += ["--dim", f"{k}={val}"]
        for flag, val in (("--nl", nl), ("--lin", lin), ("--rel", rel), ("--abs", abs_tol),
                          ("--radius0", radius0), ("--cost-stop", cost_stop)):
            if val is not None:
                cmd += [flag, repr(float(val)) if isinstance(val, float) else str(val)]
        if not precond:
            cmd.append("--noprecond")
        if materialize:
            cmd += ["--materialize", materialize]
        if force_evalj:
            cmd.append("--force-evalj")
        env = dict(os.environ)
        if threads:
            env["MINOPT_THREADS"] = str(threads)
        subprocess.run(cmd, check=True, env=env, timeout=timeout)
        return mob_read(fout)
