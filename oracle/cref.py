"""ctypes binding of the C restatement (oracle/_ref/libmo_oracle.so).

TEST INFRASTRUCTURE ONLY — the checker, never the thing measured or shipped.
Mirrors the product's Python Solver API so parity tests read the same.
"""
import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_ref", "libmo_oracle.so")


def _load():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-C", HERE, "_ref/libmo_oracle.so"], check=True, capture_output=True)
    lib = ctypes.CDLL(LIB)
    lib.moo_error.restype = ctypes.c_char_p
    lib.moo_num_cols.restype = ctypes.c_int64
    lib.moo_num_rows.restype = ctypes.c_int64
    return lib


_lib = None


class Config(ctypes.Structure):
    _fields_ = [("method", ctypes.c_int), ("nonlinear_iters", ctypes.c_int), ("linear_iters", ctypes.c_int),
                ("use_preconditioner", ctypes.c_int), ("pcg_rel_tol", ctypes.c_double),
                ("pcg_abs_tol", ctypes.c_double), ("lm_radius0", ctypes.c_double),
                ("lm_radius_min", ctypes.c_double), ("lm_radius_max", ctypes.c_double),
                ("lm_diag_min", ctypes.c_double), ("lm_diag_max", ctypes.c_double),
                ("lm_min_decrease", ctypes.c_double), ("cost_stop_tol", ctypes.c_double)]


class Result(ctypes.Structure):
    _fields_ = [("final_cost", ctypes.c_double), ("reason", ctypes.c_int), ("nonfinite_kernels", ctypes.c_int),
                ("indefinite", ctypes.c_int), ("n_trace", ctypes.c_int), ("unconstrained", ctypes.c_int64)]


class OracleError(RuntimeError):
    def __init__(self, rc, msg):
        super().__init__(f"oracle error {rc}: {msg}")
        self.rc = rc


class Oracle:
    """Sequential CPU restatement of Solver<Real> over a moplan."""

    def __init__(self, plan_text, f64=True, dims=None, cfg=None):
        global _lib
        if _lib is None:
            _lib = _load()
        self.lib = _lib
        self.dtype = np.float64 if f64 else np.float32
        h = ctypes.c_void_p()
        b = plan_text.encode()
        self._chk(self.lib.moo_create(b, len(b), int(bool(f64)), ctypes.byref(h)))
        self.h = h
        for k, v in (dims or {}).items():
            self._chk(self.lib.moo_set_dim(self.h, k.encode(), ctypes.c_int64(int(v))))
        if cfg is not None:
            c = Config()
            c.method = int(cfg.method)
            c.nonlinear_iters = cfg.nonlinear_iters
            c.linear_iters = cfg.linear_iters
            c.use_preconditioner = int(cfg.use_preconditioner)
            for k in ("pcg_rel_tol", "pcg_abs_tol", "lm_radius0", "lm_radius_min", "lm_radius_max",
                      "lm_diag_min", "lm_diag_max", "lm_min_decrease", "cost_stop_tol"):
                setattr(c, k, float(getattr(cfg, k)))
            self._chk(self.lib.moo_set_config(self.h, ctypes.byref(c)))

    def _chk(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib.moo_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.moo_destroy(self.h)
            self.h = None

    def bind(self, data):
        x = np.ascontiguousarray(data.x, self.dtype)
        self._chk(self.lib.moo_bind_x(self.h, x.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(x.size)))
        for i, a in enumerate(data.arrays):
            a = np.ascontiguousarray(a, self.dtype)
            self._chk(self.lib.moo_bind_array(self.h, i, a.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(a.size)))
        p = np.ascontiguousarray(data.params, np.float64)
        self._chk(self.lib.moo_bind_params(self.h, p.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(p.size)))
        for i, g in enumerate(data.graphs):
            v = np.ascontiguousarray(g.verts, np.uint64)
            self._chk(self.lib.moo_bind_graph(self.h, i, v.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(v.size),
                                              int(g.arity)))
        self._chk(self.lib.moo_refresh(self.h))

    def num_cols(self):
        return int(self.lib.moo_num_cols(self.h))

    def num_rows(self):
        return int(self.lib.moo_num_rows(self.h))

    def excluded(self):
        out = np.zeros(self.num_cols(), np.uint8)
        self._chk(self.lib.moo_excluded(self.h, out.ctypes.data_as(ctypes.c_void_p)))
        return out

    def cost(self):
        v = ctypes.c_double()
        self._chk(self.lib.moo_cost(self.h, ctypes.byref(v)))
        return v.value

    def residuals(self):
        out = np.zeros(self.num_rows(), self.dtype)
        self._chk(self.lib.moo_residuals(self.h, out.ctypes.data_as(ctypes.c_void_p)))
        return out

    def build_normal(self):
        b = np.zeros(self.num_cols(), self.dtype)
        m = np.zeros(self.num_cols(), self.dtype)
        self._chk(self.lib.moo_build_normal(self.h, b.ctypes.data_as(ctypes.c_void_p), m.ctypes.data_as(ctypes.c_void_p)))
        return b, m

    def apply_jtj(self, v):
        v = np.ascontiguousarray(v, self.dtype)
        out = np.zeros(self.num_cols(), self.dtype)
        self._chk(self.lib.moo_apply_jtj(self.h, v.ctypes.data_as(ctypes.c_void_p), out.ctypes.data_as(ctypes.c_void_p)))
        return out

    def solve(self):
        r = Result()
        cap = 4096
        ti = np.zeros(cap, np.int32)
        tc = np.zeros(cap)
        ta = np.zeros(cap, np.int32)
        tr = np.zeros(cap)
        tp = np.zeros(cap, np.int32)
        ptr = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        self._chk(self.lib.moo_solve(self.h, ctypes.byref(r), ptr(ti), ptr(tc), ptr(ta), ptr(tr), ptr(tp)))
        n = min(r.n_trace, cap)
        trace = dict(iter=ti[:n], cost=tc[:n], accepted=ta[:n], radius=tr[:n], pcg=tp[:n])
        return r, trace

    def get_x(self):
        out = np.zeros(self.num_cols(), self.dtype)
        self._chk(self.lib.moo_get_x(self.h, out.ctypes.data_as(ctypes.c_void_p)))
        return out

    def linearize(self):
        """linearize() (solver.hpp:291-376); returns the CSR (offs, col, val)."""
        self._chk(self.lib.moo_linearize(self.h))
        rows, nnz = ctypes.c_int64(), ctypes.c_int64()
        self._chk(self.lib.moo_jacobian(self.h, ctypes.byref(rows), ctypes.byref(nnz), None, None, None))
        offs = np.zeros(rows.value + 1, np.int64)
        col = np.zeros(nnz.value, np.int64)
        val = np.zeros(nnz.value, self.dtype)
        ptr = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        self._chk(self.lib.moo_jacobian(self.h, ctypes.byref(rows), ctypes.byref(nnz), ptr(offs), ptr(col), ptr(val)))
        return offs, col, val

    def normal_matrix(self):
        """normal_matrix() (solver.hpp:383-387) of a kJtJ plan: CSR (offs, col, val)."""
        nnz = ctypes.c_int64()
        self._chk(self.lib.moo_normal_matrix(self.h, ctypes.byref(nnz), None, None, None))
        offs = np.zeros(self.num_cols() + 1, np.int64)
        col = np.zeros(nnz.value, np.int64)
        val = np.zeros(nnz.value, self.dtype)
        ptr = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        self._chk(self.lib.moo_normal_matrix(self.h, ctypes.byref(nnz), ptr(offs), ptr(col), ptr(val)))
        return offs, col, val
