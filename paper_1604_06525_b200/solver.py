"""Python mirror of the reference solver API (minopt solver.hpp / plan.hpp).

Names, argument meaning and error behaviour follow the reference so that its
tests translate line by line:

    plan = load_plan("poisson", SolveConfig(nonlinear_iters=10))   # plan()        plan.hpp:189
    data = SolveData(x=..., arrays=[...], params=[...], graphs=[]) # SolveData     solver.hpp:23
    s = Solver(plan, data)                                         # Solver(...)   solver.hpp:84
    s.cost(); s.residuals(f); s.build_normal(); s.rhs(); s.precond()
    s.apply_jtj(v, out); r = s.solve(callback)                     # solve()       solver.hpp:389

Everything after plan() executes on the GPU through libmo_b200.so; binding
errors raise MoError with the reference Err code name (BindError,
ShapeMismatch, IndexOutOfRange, ...).
"""
import ctypes
import enum
import os
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

from . import _lib
from ._lib import MoError, call

PLAN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "plans")
ENERGY_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "energies")


class Method(enum.IntEnum):  # plan.hpp:15
    kGaussNewton = 0
    kLevenbergMarquardt = 1


class Precision(enum.IntEnum):  # plan.hpp:16
    kF32 = 0
    kF64 = 1


class StopReason(enum.IntEnum):  # solver.hpp:40-46
    kIterLimit = 0
    kCostTol = 1
    kStalled = 2
    kNonFiniteCost = 3


_REASON_NAMES = {0: "iteration_limit", 1: "cost_tolerance", 2: "stalled", 3: "nonfinite_cost"}


def to_string(r: StopReason) -> str:  # solver.hpp:48-56
    return _REASON_NAMES.get(int(r), "?")


@dataclass
class SolveConfig:  # plan.hpp:19-38 (device-relevant members)
    method: Method = Method.kGaussNewton
    precision: Precision = Precision.kF64
    nonlinear_iters: int = 8
    linear_iters: int = 100
    pcg_rel_tol: float = -1.0
    pcg_abs_tol: float = 0.0
    use_preconditioner: bool = True
    lm_radius0: float = 1e4
    lm_radius_min: float = 1e-32
    lm_radius_max: float = 1e16
    lm_diag_min: float = 1e-6
    lm_diag_max: float = 1e32
    lm_min_decrease: float = 1e-3
    cost_stop_tol: float = 0.0

    def _to_c(self):
        c = _lib.SolveConfigC()
        for name, _ in _lib.SolveConfigC._fields_:
            setattr(c, name, type(getattr(c, name))(getattr(self, name)))
        return c

    @classmethod
    def _from_c(cls, c):
        k = cls()
        for name, _ in _lib.SolveConfigC._fields_:
            setattr(k, name, getattr(c, name))
        k.method = Method(k.method)
        k.precision = Precision(k.precision)
        k.use_preconditioner = bool(k.use_preconditioner)
        return k


@dataclass
class EdgeTable:  # exec.hpp:36-43
    arity: int = 0
    verts: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))

    def size(self) -> int:
        return len(self.verts) // self.arity if self.arity else 0


@dataclass
class SolveData:  # solver.hpp:23-29
    x: np.ndarray = None
    arrays: List[np.ndarray] = field(default_factory=list)
    params: List[float] = field(default_factory=list)
    graphs: List[EdgeTable] = field(default_factory=list)


@dataclass
class IterRow:  # solver.hpp:31-38
    iter: int = 0
    cost: float = 0.0
    accepted: bool = True
    radius: float = 0.0
    pcg_iters: int = 0
    wall_ms: float = 0.0


@dataclass
class SolveResult:  # solver.hpp:58-74
    final_cost: float = 0.0
    reason: StopReason = StopReason.kIterLimit
    trace: List[IterRow] = field(default_factory=list)
    nonfinite_kernels: bool = False
    indefinite_operator: bool = False
    unconstrained: int = 0

    def trace_csv(self) -> str:
        out = ["iter,cost,accepted,radius,pcg_iters,wall_ms"]
        for r in self.trace:
            out.append(f"{r.iter},{r.cost:.17g},{int(r.accepted)},{r.radius:g},{r.pcg_iters},{r.wall_ms:g}")
        return "\n".join(out) + "\n"


class CompiledPlan:
    """A parsed moplan (the reference's CompiledPlan, plan.hpp:125-137)."""

    def __init__(self, text: str, cfg: Optional[SolveConfig] = None, dims: Optional[dict] = None,
                 exact: bool = False):
        h = ctypes.c_void_p()
        b = text.encode()
        call("mo_plan_parse", b, len(b), ctypes.byref(h))
        self._h = h
        self.text = text
        self.dims = dict(dims or {})
        self.exact = bool(exact)
        if exact:
            call("mo_plan_set_exact", self._h, 1)
        for name, extent in (dims or {}).items():
            call("mo_plan_set_dim", self._h, name.encode(), int(extent))
        if cfg is not None:
            c = cfg._to_c()
            call("mo_plan_set_config", self._h, ctypes.byref(c))
        np_, na, ng, nu = (ctypes.c_int() for _ in range(4))
        call("mo_plan_counts", self._h, ctypes.byref(np_), ctypes.byref(na), ctypes.byref(ng), ctypes.byref(nu))
        self.n_params, self.n_arrays, self.n_graphs, self.n_unknowns = np_.value, na.value, ng.value, nu.value

    @property
    def cfg(self) -> SolveConfig:
        c = _lib.SolveConfigC()
        call("mo_plan_get_config", self._h, ctypes.byref(c))
        return SolveConfig._from_c(c)

    @property
    def num_cols(self) -> int:
        n = ctypes.c_int64()
        call("mo_plan_num_cols", self._h, ctypes.byref(n))
        return n.value

    @property
    def materialize(self) -> int:
        """Materialize mode compiled into the plan (plan.hpp:17): 0 none, 1 kJ, 2 kJtJ."""
        m = ctypes.c_int()
        call("mo_plan_materialize", self._h, ctypes.byref(m))
        return m.value

    def array_size(self, i: int) -> int:
        n = ctypes.c_int64()
        call("mo_plan_array_size", self._h, i, ctypes.byref(n))
        return n.value

    def graph_arity(self, i: int) -> int:
        n = ctypes.c_int()
        call("mo_plan_graph_arity", self._h, i, ctypes.byref(n))
        return n.value

    @property
    def real_dtype(self):
        return np.float32 if self.cfg.precision == Precision.kF32 else np.float64

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.lib.mo_plan_destroy(self._h)
            self._h = None


def load_plan(name_or_path: str, cfg: Optional[SolveConfig] = None, dims: Optional[dict] = None,
              exact: bool = False) -> CompiledPlan:
    path = name_or_path
    if not os.path.exists(path):
        path = os.path.join(PLAN_DIR, name_or_path + ".moplan")
    with open(path) as f:
        return CompiledPlan(f.read(), cfg, dims, exact)


def plan(source: str, cfg: Optional[SolveConfig] = None, dims: Optional[dict] = None, materialize: int = 0,
         exact: bool = False) -> CompiledPlan:
    """plan(spec, cfg) (plan.hpp:189).  `source` is either an exported
    "moplan 1" text, or energy text / a path to a .opt file, which this
    package's own front end (frontend.py: compile_source + transform +
    schedule) turns into a plan without the reference compiler.
    `materialize` (front end only): 0 matrix-free, 1 Materialize::kJ,
    2 Materialize::kJtJ.  exact=True compiles the per-element kernels without
    FMA contraction (bitwise mode)."""
    if source.lstrip().startswith("moplan"):
        return CompiledPlan(source, cfg, dims, exact)
    from . import frontend
    if "\n" not in source and os.path.exists(source):
        with open(source) as f:
            source = f.read()
    text = frontend.plan_source(source, cfg, dims=dims, materialize=materialize)
    return CompiledPlan(text, cfg, None, exact)


def _as(a, dtype):
    return np.ascontiguousarray(np.asarray(a, dtype=dtype))


class Solver:
    """minopt::Solver<Real> (solver.hpp:80-635) over the device session."""

    def __init__(self, plan_: CompiledPlan, data: SolveData, device: int = 0, comm=None, rows=None, halo=0):
        """comm/rows: strip shard owning axis-0 rows [rows[0], rows[1]) of the
        plan's grid domain (see sharded.py); `data` is then the strip's LOCAL
        data (its stored rows [lo, hi), halos included)."""
        self.plan = plan_
        self.data = data
        self.dtype = plan_.real_dtype
        self._comm = comm
        h = ctypes.c_void_p()
        if comm is None:
            call("mo_session_create", plan_._h, int(device), ctypes.byref(h))
        else:
            call("mo_session_create_shard_halo", plan_._h, int(device), comm, int(rows[0]), int(rows[1]), int(halo),
                 ctypes.byref(h))
        self._h = h
        self._bind_all()
        call("mo_refresh", self._h)

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.lib.mo_session_destroy(self._h)
            self._h = None

    # -- binding (SolveData -> device) --------------------------------------
    def _bind_all(self):
        d = self.data
        if d.x is None:
            raise MoError(15, "unknown vector size does not match the plan layout")
        x = _as(d.x, self.dtype)
        call("mo_bind_x", self._h, x.ctypes.data, x.size)
        if len(d.arrays) != self.plan.n_arrays:
            raise MoError(15, "array count does not match the declaration")
        for i, a in enumerate(d.arrays):
            a = _as(a, self.dtype)
            call("mo_bind_array", self._h, i, a.ctypes.data, a.size)
        p = _as(d.params, np.float64)
        call("mo_bind_params", self._h, p.ctypes.data, p.size)
        if len(d.graphs) != self.plan.n_graphs:
            raise MoError(15, "graph count does not match the declaration")
        for i, g in enumerate(d.graphs):
            v = _as(g.verts, np.uint64)
            call("mo_bind_graph", self._h, i, v.ctypes.data, v.size, int(g.arity))

    def refresh(self):
        call("mo_refresh", self._h)

    # -- reference routines ---------------------------------------------------
    def num_cols(self) -> int:
        n = ctypes.c_int64()
        call("mo_num_cols", self._h, ctypes.byref(n))
        return n.value

    def num_rows(self) -> int:
        n = ctypes.c_int64()
        call("mo_num_rows", self._h, ctypes.byref(n))
        return n.value

    def excluded(self) -> np.ndarray:
        out = np.zeros(self.num_cols(), np.uint8)
        call("mo_get_excluded", self._h, out.ctypes.data, out.size)
        return out

    def cost(self) -> float:
        v = ctypes.c_double()
        call("mo_cost", self._h, ctypes.byref(v))
        return v.value

    def residuals(self, f: Optional[np.ndarray] = None) -> np.ndarray:
        n = self.num_rows()
        if f is not None and (f.size != n or f.dtype != self.dtype):
            raise MoError(10, "residual vector size does not match the instance count")
        out = np.empty(n, self.dtype) if f is None else f
        call("mo_residuals", self._h, out.ctypes.data, n)
        return out

    def build_normal(self):
        call("mo_build_normal", self._h)

    def rhs(self) -> np.ndarray:
        out = np.empty(self.num_cols(), self.dtype)
        call("mo_get_rhs", self._h, out.ctypes.data, out.size)
        return out

    def precond(self) -> np.ndarray:
        out = np.empty(self.num_cols(), self.dtype)
        call("mo_get_precond", self._h, out.ctypes.data, out.size)
        return out

    def apply_jtj(self, v, out: Optional[np.ndarray] = None) -> np.ndarray:
        v = _as(v, self.dtype)
        if v.size != self.num_cols():
            raise MoError(10, "apply_jtj(): vector size mismatch")
        if out is not None and (not isinstance(out, np.ndarray) or out.dtype != self.dtype
                                or out.size != v.size or not out.flags.c_contiguous or not out.flags.writeable):
            raise MoError(10, "apply_jtj(): out must be a writable C-contiguous vector of num_cols Reals")
        res = np.empty(v.size, self.dtype) if out is None else out
        call("mo_apply_jtj", self._h, v.ctypes.data, res.ctypes.data, v.size)
        return res

    def linearize(self) -> None:
        """linearize() (solver.hpp:291-377): Jacobian lanes at x, on the device.
        Materialize::kJ sessions apply 2 J^T J v from them afterwards."""
        call("mo_linearize", self._h)

    def jacobian(self):
        """jacobian() (solver.hpp:378-381) as CSR arrays (offs, col, val) in the
        reference's row and column order."""
        rows, cols, nnz = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        call("mo_jacobian_size", self._h, ctypes.byref(rows), ctypes.byref(cols), ctypes.byref(nnz))
        offs = np.empty(rows.value + 1, np.int64)
        col = np.empty(nnz.value, np.int64)
        val = np.empty(nnz.value, self.dtype)
        call("mo_get_jacobian", self._h, offs.ctypes.data, col.ctypes.data, val.ctypes.data, nnz.value)
        return offs, col, val

    def normal_matrix(self):
        """normal_matrix() (solver.hpp:383-387) of a kJtJ session: CSR (offs, col, val)."""
        nnz = ctypes.c_int64()
        call("mo_normal_matrix_size", self._h, ctypes.byref(nnz))
        offs = np.empty(self.num_cols() + 1, np.int64)
        col = np.empty(nnz.value, np.int64)
        val = np.empty(nnz.value, self.dtype)
        call("mo_get_normal_matrix", self._h, offs.ctypes.data, col.ctypes.data, val.ctypes.data, nnz.value)
        return offs, col, val

    def saw_nonfinite_kernel(self) -> bool:
        v = ctypes.c_int()
        call("mo_saw_nonfinite", self._h, ctypes.byref(v))
        return bool(v.value)

    def get_x(self) -> np.ndarray:
        out = np.empty(self.num_cols(), self.dtype)
        call("mo_get_x", self._h, out.ctypes.data, out.size)
        return out

    def solve(self, callback: Optional[Callable[[int, SolveData], None]] = None) -> SolveResult:
        """solve(callback) (solver.hpp:389-515); updates data.x in place."""
        err = []

        def tramp(it, _s, _u):
            try:
                self.data.x = self.get_x()
                callback(it, self.data)
                self._bind_all()
            except Exception as e:  # surfaced after mo_solve returns
                err.append(e)

        cb = _lib.ITER_CB(tramp) if callback else _lib.ITER_CB()
        res = _lib.SolveResultC()
        call("mo_solve", self._h, cb, None, ctypes.byref(res))
        if err:
            raise err[0]
        out = SolveResult(
            final_cost=res.final_cost, reason=StopReason(res.reason),
            nonfinite_kernels=bool(res.nonfinite_kernels), indefinite_operator=bool(res.indefinite_operator),
            unconstrained=int(res.unconstrained))
        for i in range(res.n_trace):
            r = res.trace[i]
            out.trace.append(IterRow(r.iter, r.cost, bool(r.accepted), r.radius, r.pcg_iters, r.wall_ms))
        x = self.get_x()
        if isinstance(self.data.x, np.ndarray) and self.data.x.dtype == x.dtype and self.data.x.size == x.size:
            self.data.x[...] = x
        else:
            self.data.x = x
        return out

    # -- measurement hooks ----------------------------------------------------
    def set_profiling(self, on: bool):
        call("mo_set_profiling", self._h, int(bool(on)))

    def profile(self, kind: int):
        ms, n = ctypes.c_double(), ctypes.c_int64()
        call("mo_profile_read", self._h, int(kind), ctypes.byref(ms), ctypes.byref(n))
        return ms.value, n.value

    def profile_reset(self):
        call("mo_profile_reset", self._h)

    def bench_kernel(self, which: int = 0, reps: int = 20) -> float:
        """ms per launch of the J^T J p apply (which=0) or build_normal (1):
        `reps` launches replayed as one CUDA graph, best of 3 (mo_bench_kernel;
        clobbers the PCG scratch vectors)."""
        ms = ctypes.c_double()
        call("mo_bench_kernel", self._h, int(which), int(reps), ctypes.byref(ms))
        return ms.value

    def apply_kernel(self, gather_set: int = 0) -> str:
        """Name of the J^T J p kernel the session runs for a gather set."""
        buf = ctypes.create_string_buffer(128)
        call("mo_apply_kernel", self._h, int(gather_set), buf, 128)
        return buf.value.decode()

    def normal_kernel(self, gather_set: int = 0) -> str:
        """Name of the build_normal (J^T F + Jacobi) kernel of a gather set."""
        buf = ctypes.create_string_buffer(128)
        call("mo_normal_kernel", self._h, int(gather_set), buf, 128)
        return buf.value.decode()

    def kernel_launches(self) -> int:
        n = ctypes.c_int64()
        call("mo_kernel_launches", self._h, ctypes.byref(n))
        return n.value


@dataclass
class PcgOutcome:
    """PcgOutcome (pcg.hpp:19-24)."""
    iterations: int = 0
    indefinite: bool = False
    nonfinite: bool = False


def pcg(apply, b, m, max_iters: int = 10, tol_rel: float = 1e-3, tol_abs: float = 0.0,
        use_preconditioner: bool = True, excluded=None, device: int = 0):
    """pcg<Real>(apply_a, b, m, delta, opt, ws, excluded) (pcg.hpp:59-130) on
    the device, defaults of PcgOptions (pcg.hpp:12-17).  `apply(x, y, stream)`
    receives device pointers (int) of len(b) Reals and must leave y = A x
    complete on return (or enqueued on the cudaStream_t `stream`).  Real is
    b's dtype (float32 / float64).  Returns (delta, PcgOutcome)."""
    b = np.ascontiguousarray(b)
    dt = np.float32 if b.dtype == np.float32 else np.float64
    b = b.astype(dt, copy=False)
    m = _as(m, dt)
    if m.size != b.size:
        raise MoError(10, "pcg operand sizes do not match")
    delta = np.zeros(b.size, dt)
    ex = None if excluded is None else np.ascontiguousarray(excluded, np.uint8)
    if ex is not None and ex.size != b.size:
        raise MoError(10, "pcg operand sizes do not match")
    err = []

    def tramp(x, y, stream, _user):
        try:
            apply(x, y, stream)
        except Exception as e:  # surfaced after mo_pcg returns
            err.append(e)

    cb = _lib.APPLY_FN(tramp)
    opt = _lib.PcgOptionsC(int(max_iters), float(tol_rel), float(tol_abs), int(bool(use_preconditioner)))
    out = _lib.PcgOutcomeC()
    call("mo_pcg", int(device), 0 if dt == np.float32 else 1, b.size, cb, None, b.ctypes.data, m.ctypes.data,
         delta.ctypes.data, ctypes.byref(opt), None if ex is None else ex.ctypes.data, ctypes.byref(out))
    if err:
        raise err[0]
    return delta, PcgOutcome(out.iterations, bool(out.indefinite), bool(out.nonfinite))
