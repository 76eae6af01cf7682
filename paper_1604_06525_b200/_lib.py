"""ctypes binding of libmo_b200.so (include/mo_b200.h).

The library is built in-tree (``python __graft_entry__.py`` or
``make -C paper_1604_06525_b200/csrc``).  It is loaded on first use; there is
no fallback: any call without the built library raises ImportError.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmo_b200.so")

_LIB = None


def _load():
    """dlopen libmo_b200.so on first use (not at package import, so that
    importing the workload generators does not map the product library into
    processes that never call it, e.g. bench.py's reference arm).  A missing
    library raises: there is no CPU fallback."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make -C {_HERE}/csrc` "
                "(the B200 solver has no CPU fallback)")
        lib_ = ctypes.CDLL(LIB_PATH)
        for _name, (_res, _args) in SIGNATURES.items():
            _f = getattr(lib_, _name)
            _f.restype = _res
            _f.argtypes = _args
        _LIB = lib_
    return _LIB


def __getattr__(name):  # `_lib.lib` loads the library lazily (PEP 562)
    if name == "lib":
        return _load()
    raise AttributeError(name)

c_int, c_int64, c_double, c_void_p, c_char_p, c_size_t = (
    ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p, ctypes.c_char_p, ctypes.c_size_t)


class SolveConfigC(ctypes.Structure):
    _fields_ = [("method", c_int), ("precision", c_int), ("nonlinear_iters", c_int),
                ("linear_iters", c_int), ("pcg_rel_tol", c_double), ("pcg_abs_tol", c_double),
                ("use_preconditioner", c_int), ("lm_radius0", c_double), ("lm_radius_min", c_double),
                ("lm_radius_max", c_double), ("lm_diag_min", c_double), ("lm_diag_max", c_double),
                ("lm_min_decrease", c_double), ("cost_stop_tol", c_double)]


class IterRowC(ctypes.Structure):
    _fields_ = [("iter", c_int), ("cost", c_double), ("accepted", c_int), ("radius", c_double),
                ("pcg_iters", c_int), ("wall_ms", c_double)]


class SolveResultC(ctypes.Structure):
    _fields_ = [("final_cost", c_double), ("reason", c_int), ("nonfinite_kernels", c_int),
                ("indefinite_operator", c_int), ("unconstrained", c_int64), ("n_trace", c_int),
                ("trace", ctypes.POINTER(IterRowC))]


ITER_CB = ctypes.CFUNCTYPE(None, c_int, c_void_p, c_void_p)
APPLY_FN = ctypes.CFUNCTYPE(None, c_void_p, c_void_p, c_void_p, c_void_p)


class PcgOptionsC(ctypes.Structure):
    _fields_ = [("max_iters", c_int), ("tol_rel", c_double), ("tol_abs", c_double), ("use_preconditioner", c_int)]


class PcgOutcomeC(ctypes.Structure):
    _fields_ = [("iterations", c_int), ("indefinite", c_int), ("nonfinite", c_int)]

# Every symbol include/mo_b200.h declares, with its argument types.
SIGNATURES = {
    "mo_last_error": (c_char_p, []),
    "mo_version": (c_char_p, []),
    "mo_device_count": (c_int, [ctypes.POINTER(c_int)]),
    "mo_plan_parse": (c_int, [c_char_p, c_size_t, ctypes.POINTER(c_void_p)]),
    "mo_plan_set_dim": (c_int, [c_void_p, c_char_p, c_int64]),
    "mo_plan_get_config": (c_int, [c_void_p, ctypes.POINTER(SolveConfigC)]),
    "mo_plan_set_config": (c_int, [c_void_p, ctypes.POINTER(SolveConfigC)]),
    "mo_plan_num_cols": (c_int, [c_void_p, ctypes.POINTER(c_int64)]),
    "mo_plan_precompile": (c_int, [c_void_p, c_int]),
    "mo_plan_set_exact": (c_int, [c_void_p, c_int]),
    "mo_plan_counts": (c_int, [c_void_p] + [ctypes.POINTER(c_int)] * 4),
    "mo_plan_array_size": (c_int, [c_void_p, c_int, ctypes.POINTER(c_int64)]),
    "mo_plan_graph_arity": (c_int, [c_void_p, c_int, ctypes.POINTER(c_int)]),
    "mo_plan_destroy": (None, [c_void_p]),
    "mo_session_create": (c_int, [c_void_p, c_int, ctypes.POINTER(c_void_p)]),
    "mo_session_destroy": (None, [c_void_p]),
    "mo_bind_x": (c_int, [c_void_p, c_void_p, c_int64]),
    "mo_bind_array": (c_int, [c_void_p, c_int, c_void_p, c_int64]),
    "mo_bind_params": (c_int, [c_void_p, c_void_p, c_int64]),
    "mo_bind_graph": (c_int, [c_void_p, c_int, c_void_p, c_int64, c_int]),
    "mo_bind_x_device": (c_int, [c_void_p, c_void_p, c_int64]),
    "mo_bind_array_device": (c_int, [c_void_p, c_int, c_void_p, c_int64]),
    "mo_refresh": (c_int, [c_void_p]),
    "mo_num_cols": (c_int, [c_void_p, ctypes.POINTER(c_int64)]),
    "mo_num_rows": (c_int, [c_void_p, ctypes.POINTER(c_int64)]),
    "mo_get_excluded": (c_int, [c_void_p, c_void_p, c_int64]),
    "mo_cost": (c_int, [c_void_p, ctypes.POINTER(c_double)]),
    "mo_residuals": (c_int, [c_void_p, c_void_p, c_int64]),
    "mo_build_normal": (c_int, [c_void_p]),
    "mo_get_rhs": (c_int, [c_void_p, c_void_p, c_int64]),
    "mo_get_precond": (c_int, [c_void_p, c_void_p, c_int64]),
    "mo_apply_jtj": (c_int, [c_void_p, c_void_p, c_void_p, c_int64]),
    "mo_apply_jtj_device": (c_int, [c_void_p, c_void_p, c_void_p]),
    "mo_solve": (c_int, [c_void_p, ITER_CB, c_void_p, ctypes.POINTER(SolveResultC)]),
    "mo_get_x": (c_int, [c_void_p, c_void_p, c_int64]),
    "mo_saw_nonfinite": (c_int, [c_void_p, ctypes.POINTER(c_int)]),
    "mo_plan_halo_rows": (c_int, [c_void_p, ctypes.POINTER(c_int)]),
    "mo_nccl_unique_id": (c_int, [c_void_p, c_size_t]),
    "mo_comm_create_nccl": (c_int, [c_void_p, c_size_t, c_int, c_int, c_int, ctypes.POINTER(c_void_p)]),
    "mo_world_create_local": (c_int, [c_int, c_int, ctypes.POINTER(c_void_p)]),
    "mo_comm_create_local": (c_int, [c_void_p, c_int, ctypes.POINTER(c_void_p)]),
    "mo_world_destroy": (None, [c_void_p]),
    "mo_comm_destroy": (None, [c_void_p]),
    "mo_session_create_shard": (c_int, [c_void_p, c_int, c_void_p, c_int64, c_int64, ctypes.POINTER(c_void_p)]),
    "mo_session_create_shard_halo": (c_int, [c_void_p, c_int, c_void_p, c_int64, c_int64, c_int,
                                             ctypes.POINTER(c_void_p)]),
    "mo_session_local_layout": (c_int, [c_void_p] + [ctypes.POINTER(c_int64)] * 4),
    "mo_set_profiling": (c_int, [c_void_p, c_int]),
    "mo_profile_read": (c_int, [c_void_p, c_int, ctypes.POINTER(c_double), ctypes.POINTER(c_int64)]),
    "mo_profile_reset": (c_int, [c_void_p]),
    "mo_bench_kernel": (c_int, [c_void_p, c_int, c_int, ctypes.POINTER(ctypes.c_double)]),
    "mo_optd_stat": (c_int, [c_char_p, ctypes.POINTER(c_int), ctypes.POINTER(c_int), ctypes.POINTER(c_int),
                             ctypes.POINTER(c_int64), c_int]),
    "mo_optd_read": (c_int, [c_char_p, c_void_p, c_int64, c_int]),
    "mo_optd_write": (c_int, [c_char_p, c_int, c_int, c_int, ctypes.POINTER(c_int64), c_void_p]),
    "mo_optg_stat": (c_int, [c_char_p, ctypes.POINTER(c_int), ctypes.POINTER(c_int64)]),
    "mo_optg_read": (c_int, [c_char_p, ctypes.POINTER(ctypes.c_uint64), c_int64]),
    "mo_optg_write": (c_int, [c_char_p, c_int, c_int64, ctypes.POINTER(ctypes.c_uint64)]),
    "mo_session_stream": (c_int, [c_void_p, ctypes.POINTER(c_void_p)]),
    "mo_kernel_launches": (c_int, [c_void_p, ctypes.POINTER(c_int64)]),
    "mo_apply_kernel": (c_int, [c_void_p, c_int, ctypes.c_char_p, ctypes.c_size_t]),
    "mo_normal_kernel": (c_int, [c_void_p, c_int, ctypes.c_char_p, ctypes.c_size_t]),
    "mo_plan_materialize": (c_int, [c_void_p, ctypes.POINTER(c_int)]),
    "mo_pcg": (c_int, [c_int, c_int, c_int64, APPLY_FN, c_void_p, c_void_p, c_void_p, c_void_p,
                       ctypes.POINTER(PcgOptionsC), c_void_p, ctypes.POINTER(PcgOutcomeC)]),
    "mo_linearize": (c_int, [c_void_p]),
    "mo_jacobian_size": (c_int, [c_void_p] + [ctypes.POINTER(c_int64)] * 3),
    "mo_get_jacobian": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64]),
    "mo_normal_matrix_size": (c_int, [c_void_p, ctypes.POINTER(c_int64)]),
    "mo_get_normal_matrix": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64]),
}


# minopt::Err names (common.hpp:13-32), indexed by ABI code - 1.
ERR_NAMES = ["SyntaxError", "UndeclaredIdentifier", "ArityMismatch", "NonConstantOffset",
             "MixedDomain", "NonConstantExponent", "DomainMismatch", "NonBooleanPredicate",
             "CyclicComputedArray", "ShapeMismatch", "IndexOutOfRange", "FormatError",
             "TruncatedFile", "GraphDomainError", "BindError", "NonFiniteCost", "CyclicIR",
             "InternalError"]


class MoError(RuntimeError):
    """Mirror of minopt::Error: carries the reference Err code name in `.code`."""

    def __init__(self, rc, msg):
        if 1 <= rc <= len(ERR_NAMES):
            code = ERR_NAMES[rc - 1]
        elif rc == 101:
            code = "CudaError"
        elif rc == 102:
            code = "NoDevice"
        else:
            code = f"Error{rc}"
        super().__init__(f"{code}: {msg}")
        self.code = code
        self.rc = rc


def call(name, *args):
    lib = _load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        raise MoError(rc, lib.mo_last_error().decode(errors="replace"))
    return rc


def device_count():
    n = c_int(0)
    call("mo_device_count", ctypes.byref(n))
    return n.value
