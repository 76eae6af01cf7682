"""B200-native matrix-free Gauss-Newton / Levenberg-Marquardt core of Opt
(arXiv 1604.06525): a drop-in device implementation of the reference minopt
solver path (cost, J^T F + Jacobi, matrix-free J^T J p, Jacobi PCG, GN/LM).
"""
from ._lib import MoError, device_count
from .solver import (CompiledPlan, EdgeTable, IterRow, Method, PcgOutcome, Precision, SolveConfig, SolveData,
                     SolveResult, Solver, StopReason, load_plan, pcg, plan, to_string)

__all__ = ["MoError", "device_count", "CompiledPlan", "EdgeTable", "IterRow", "Method", "Precision",
           "SolveConfig", "SolveData", "SolveResult", "Solver", "StopReason", "load_plan", "plan",
           "to_string", "pcg", "PcgOutcome"]
