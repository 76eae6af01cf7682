"""Shared test helpers: golden-case loading and tolerance checks."""
import json
import os

import numpy as np

from paper_1604_06525_b200 import EdgeTable, Method, Precision, SolveConfig, SolveData, load_plan

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden_names(prefix=""):
    return sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz") and f.startswith(prefix))


def cfg_from(d, prec):
    c = SolveConfig()
    c.precision = Precision.kF32 if prec == "f32" else Precision.kF64
    if d.get("method") == "lm":
        c.method = Method.kLevenbergMarquardt
    for k, attr in (("nl", "nonlinear_iters"), ("lin", "linear_iters"), ("rel", "pcg_rel_tol"),
                    ("radius0", "lm_radius0"), ("cost_stop", "cost_stop_tol")):
        if d.get(k) is not None:
            setattr(c, attr, type(getattr(c, attr))(d[k]))
    return c


class Golden:
    def __init__(self, name):
        self.name = name
        z = np.load(os.path.join(GOLDEN, name + ".npz"))
        self.z = {k: z[k] for k in z.files}
        self.prec = str(self.z["prec"])
        self.dtype = np.float32 if self.prec == "f32" else np.float64
        self.cfg_dict = json.loads(str(self.z["cfg"]))
        self.cfg = cfg_from(self.cfg_dict, self.prec)
        self.cmds = str(self.z["cmds"]).split(",")

    def plan(self, exact=False):
        return load_plan(os.path.join(GOLDEN, self.name + ".moplan"), self.cfg, exact=exact)

    def data(self):
        z = self.z
        return SolveData(
            x=z["x"].astype(self.dtype),
            arrays=[z[f"array{i}"].astype(self.dtype) for i in range(int(z["n_arrays"]))],
            params=list(z["params"]),
            graphs=[EdgeTable(int(z[f"graph{i}_arity"]), z[f"graph{i}"].astype(np.uint64))
                    for i in range(int(z["n_graphs"]))])

    def ref(self, key):
        return self.z.get("ref_" + key)


def assert_close_vec(got, ref, rel, what="", floor=False):
    """Per-element check |got-ref| <= rel*|ref| (north_star: 1e-5 fp32,
    1e-10 fp64 per element).

    floor=True adds an absolute floor rel*max|ref| (||ref||_inf): only for
    outputs that are sums of cancelling terms (2 J^T J v, b = -2 J^T F,
    residual differences, J / H entries, x after a solve), where an element
    that is exactly or nearly zero in the reference is a rounding residue of
    O(||ref||_inf) terms and has no relative accuracy to check.  Strictly
    positive sums without cancellation (m = diag 2 J^T J) use floor=False."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    assert got.shape == ref.shape, f"{what}: shape {got.shape} vs {ref.shape}"
    scale = np.max(np.abs(ref)) if (ref.size and floor) else 0.0
    tol = rel * np.abs(ref) + rel * scale + 1e-300
    bad = np.abs(got - ref) > tol
    bad &= ~(np.isnan(got) & np.isnan(ref))
    if bad.any():
        i = int(np.argmax(np.abs(got - ref) - tol))
        raise AssertionError(f"{what}: {bad.sum()} of {got.size} elements differ; worst at {i}: "
                             f"got {got[i]!r} ref {ref[i]!r} (rel {rel}, floor {floor})")


def rel_close(a, b, rel):
    if np.isnan(a) and np.isnan(b):
        return True
    if np.isinf(a) or np.isinf(b):
        return a == b
    return abs(a - b) <= rel * max(abs(a), abs(b), 1e-300)
