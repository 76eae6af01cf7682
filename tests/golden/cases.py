"""Golden cases: the reference's own unit tests for the solver path
(reference proj/tests/test_solver.cpp, test_transform.cpp, test_exec.cpp) plus
small instances of the five BASELINE configs.  make_golden.py runs each case
through the UNMODIFIED reference (oracle/_ref/ref_driver) and the plan
exporter (integration/_build/export_plan) and stores the results here as
<name>.moplan + <name>.npz, so GPU tests never need /root/reference.
"""
import numpy as np

K_CHAIN = """dim W 2
unknown X [W]
array A [W]
energy X(0) - A(0)
energy X(0) - X(1)
"""

# test_solver.cpp:103-153 (materialized-vs-free energy; we check the free side)
K_SINCHAIN = """dim W 9
unknown X [W]
array A [W]
energy sin(X(0)) - A(0)
energy 0.5 * (X(0) - X(1))
"""

K_GRAPH = "dim N 2\nunknown P [N]\ngraph G (a, b)\nenergy P(G.a) - P(G.b)\n"
K_GRAPH1 = "dim N 2\nunknown P [N]\ngraph G (a, b)\nenergy P(G.a) - P(G.b) + 1\n"
K_EXCL = "dim W 2\nunknown X [W]\narray A [W]\nenergy X(0) - A(0)\nexclude less(index(0), 1)\n"
K_INLINED = "dim W 5\nunknown X [W]\narray A [W]\nenergy sin(X(0)) - A(0)\n"
K_CACHED = "dim W 5\nunknown X [W]\narray A [W]\ncomputed S cache = sin(X(0))\nenergy S(0) - A(0)\n"
K_FREEZE = "dim W 3\nunknown X [W]\ncomputed S freeze = X(0) * X(0)\nenergy S(0) - X(0)\n"
K_FLAT = "dim W 2\nunknown X [W]\narray A [W]\nenergy A(0)\n"
K_LOG = "dim W 1\nunknown X [W]\nenergy log(X(0))\n"
K_UNCON = "dim W 2\nunknown X [W]\nunknown Y [W]\narray A [W]\nenergy X(0) - A(0)\n"
K_EMPTY = "dim W 3\nunknown X [W]\n"
# test_transform.cpp:208-286 dense-Jacobian oracle energy
K_DENSE = """dim W 4
dim H 3
unknown X [W, H]
array A [W, H]
energy select(inbounds(1, 0), X(1, 0) - X(0, 0), 0) + 0.5 * (X(0, 0) - A(0, 0))
energy select(inbounds(0, 1), 2 * X(0, 1) - X(0, 0), 0)
"""
# extra coverage: pow / abs / cos / exp / atan / comparisons / 3-D domain / arity-3 graph
K_OPS = """dim W 6
dim H 5
param w
unknown X [W, H] : 2
array A [W, H]
energy select(greater(A(0,0), 0.3), w * (X(0,0)[0] * X(0,0)[0] - A(0,0)), X(0,0)[1] - cos(A(0,0)))
energy pow(X(0,0)[0], 3) - 0.5 * exp(X(-1,0)[1] * 0.25) + atan(X(0,1)[0])
energy abs(X(0,0)[1] - X(1,1)[0]) + sqrt(X(0,0)[0] * X(0,0)[0] + 1)
"""
K_VOL = """dim A 4
dim B 3
dim C 5
unknown U [A, B, C]
array T [A, B, C]
energy U(0,0,0) - U(1,0,0) - T(0,0,0)
energy U(0,0,0) - U(0,0,-1) + 0.25 * U(0,1,0)
"""
K_TRI = """dim N 5
unknown P [N] : 2
array Q [N]
graph G (a, b, c)
energy P(G.a) - 0.5 * (P(G.b) + P(G.c)) + vec(Q(G.a), 0)
energy select(greater(Q(G.b), 0.5), sin(P(G.b)[0]) - P(G.c)[1], 0)
"""


def _r(seed, n, lo=-1.0, hi=1.0):
    return list(np.random.default_rng(seed).uniform(lo, hi, n))


def unit_cases():
    """name -> dict(src, x, arrays, params, graphs, cfg(dict), prec, cmds, v)."""
    C = {}
    C["chain"] = dict(src=K_CHAIN, x=[0.0, 0.0], arrays=[[1.0, 0.0]], cfg=dict(nl=1),
                      cmds=["cost", "residuals", "normal", "jtj", "solve"], v=[1.0, 0.0])
    C["chain_f32"] = dict(C["chain"], prec="f32")
    C["sinchain"] = dict(src=K_SINCHAIN, x=_r(41, 9), arrays=[_r(42, 9)],
                         cmds=["cost", "residuals", "normal", "jtj", "solve"], v=_r(43, 9))
    C["graph"] = dict(src=K_GRAPH, x=[3.0, 1.0], graphs=[(2, [0, 1])],
                      cmds=["cost", "residuals", "normal", "jtj", "solve"], v=[1.0, 0.0])
    C["graph_degenerate"] = dict(src=K_GRAPH1, x=[5.0, 7.0], graphs=[(2, [0, 0])],
                                 cmds=["cost", "normal", "jtj"], v=[1.0, 0.0])
    C["exclude"] = dict(src=K_EXCL, x=[-0.0, 0.0], arrays=[[1.0, 2.0]], cfg=dict(nl=1),
                        cmds=["cost", "normal", "jtj", "solve"], v=[1.0, 1.0])
    x5, a5 = _r(7, 5, -2, 2), _r(8, 5, -2, 2)
    C["inlined"] = dict(src=K_INLINED, x=x5, arrays=[a5], cmds=["cost", "normal", "jtj", "solve"], v=_r(9, 5, -2, 2))
    C["cached"] = dict(C["inlined"], src=K_CACHED)
    C["freeze"] = dict(src=K_FREEZE, x=[2.0, 3.0, 4.0], cmds=["cost", "normal", "jtj"], v=[1.0, 0.5, -1.0])
    C["lm_quadratic"] = dict(src=K_CHAIN, x=[0.0, 0.0], arrays=[[1.0, 0.0]], cfg=dict(nl=2, method="lm"),
                             cmds=["solve"])
    C["lm_flat"] = dict(src=K_FLAT, x=[0.25, -0.75], arrays=[[3.0, 4.0]], cfg=dict(method="lm"), cmds=["solve"])
    C["gn_flat"] = dict(src=K_FLAT, x=[0.25, -0.75], arrays=[[3.0, 4.0]], cfg=dict(nl=3), cmds=["solve"])
    C["nan_start"] = dict(src=K_LOG, x=[-1.0], cmds=["solve"])
    C["nan_gn_step"] = dict(src=K_LOG, x=[4.0], cmds=["solve"])
    C["nan_lm_recover"] = dict(src=K_LOG, x=[4.0], cfg=dict(method="lm", radius0=1e8, nl=20), cmds=["solve"])
    C["unconstrained"] = dict(src=K_UNCON, x=[0.0, 0.0, 41.5, -2.25], arrays=[[1.0, 2.0]], cfg=dict(nl=1),
                              cmds=["normal", "solve"])
    C["cost_stop"] = dict(src=K_CHAIN, x=[0.0, 0.0], arrays=[[1.0, 0.0]], cfg=dict(nl=8, cost_stop=1e-12),
                          cmds=["solve"])
    C["empty"] = dict(src=K_EMPTY, x=[1.0, 2.0, 3.0], cfg=dict(nl=1), cmds=["cost", "solve"])
    C["dense"] = dict(src=K_DENSE, x=_r(31, 12, -2, 2), arrays=[_r(32, 12, -2, 2)], cfg=dict(nl=1),
                      cmds=["cost", "residuals", "normal", "jtj", "solve"], v=_r(33, 12, -2, 2))
    C["ops"] = dict(src=K_OPS, x=_r(51, 60, 0.1, 1.0), arrays=[_r(52, 30, 0, 1)], params=[1.5],
                    cfg=dict(nl=3, lin=8), cmds=["cost", "residuals", "normal", "jtj", "solve"], v=_r(53, 60))
    C["ops_f32"] = dict(C["ops"], prec="f32")
    C["volume"] = dict(src=K_VOL, x=_r(61, 60), arrays=[_r(62, 60)], cfg=dict(nl=2),
                       cmds=["cost", "residuals", "normal", "jtj", "solve"], v=_r(63, 60))
    C["tri_graph"] = dict(src=K_TRI, x=_r(71, 10), arrays=[_r(72, 5, 0, 1)],
                          graphs=[(3, [0, 1, 2, 1, 2, 3, 4, 0, 2, 2, 2, 4, 3, 3, 1])], cfg=dict(nl=3, lin=6),
                          cmds=["cost", "residuals", "normal", "jtj", "solve"], v=_r(73, 10))
    # Materialize::kJ (solver.hpp:278-376) and force_evalj linearize / jacobian
    # (test_solver.cpp:39-77, 103-153, 186-204)
    lin = ["cost", "normal", "linearize", "jtj", "solve"]
    C["mat_chain_lanes"] = dict(C["chain"], cfg=dict(nl=1, force_evalj=True), cmds=["normal", "jtj", "linearize"])
    C["mat_sinchain"] = dict(C["sinchain"], cfg=dict(materialize="j"), cmds=lin)
    C["mat_sinchain_lm"] = dict(C["sinchain"], cfg=dict(materialize="j", method="lm", nl=4), cmds=lin)
    C["mat_graph_degenerate"] = dict(C["graph_degenerate"], cfg=dict(materialize="j"), cmds=["cost", "linearize", "jtj", "solve"])
    C["mat_exclude"] = dict(C["exclude"], cfg=dict(nl=1, materialize="j"), cmds=lin)
    C["mat_dense"] = dict(C["dense"], cfg=dict(nl=1, materialize="j"), cmds=lin)
    C["mat_ops"] = dict(C["ops"], cfg=dict(nl=3, lin=8, materialize="j"), cmds=lin)
    C["mat_ops_f32"] = dict(C["mat_ops"], prec="f32")
    C["mat_volume"] = dict(C["volume"], cfg=dict(nl=2, materialize="j"), cmds=lin)
    C["mat_tri_graph"] = dict(C["tri_graph"], cfg=dict(nl=3, lin=6, materialize="j"), cmds=lin)
    C["mat_cached"] = dict(C["cached"], cfg=dict(materialize="j"), cmds=lin)  # cache-mode computed array
    C["mat_freeze"] = dict(C["freeze"], cfg=dict(materialize="j"), cmds=["cost", "normal", "linearize", "jtj"])
    # Materialize::kJtJ (H = 2 J^T J assembled, solver.hpp:370-374)
    for k in ("sinchain", "sinchain_lm", "graph_degenerate", "exclude", "dense", "ops", "ops_f32", "volume",
              "tri_graph", "cached", "freeze"):
        c = dict(C["mat_" + k])
        c["cfg"] = dict(c["cfg"], materialize="jtj")
        C["math_" + k] = c
    for c in C.values():
        c.setdefault("arrays", [])
        c.setdefault("params", [])
        c.setdefault("graphs", [])
        c.setdefault("cfg", {})
        c.setdefault("prec", "f64")
        c.setdefault("v", None)
    return C


# Small instances of the BASELINE configs: (workload fn, kwargs, cfg)
CONFIG_CASES = {
    "cfg_poisson": ("poisson", dict(W=24, H=20), dict(nl=3, lin=10, rel=0.0)),
    "cfg_arap_warp": ("arap_warp", dict(W=24, H=20, nhandles=6), dict(nl=3, lin=10, rel=0.0)),
    "cfg_sfs": ("sfs", dict(W=24, H=18), dict(nl=3, lin=10, rel=0.0, method="lm")),
    "cfg_arap_mesh": ("arap_mesh", dict(n=8, nhandles=5), dict(nl=3, lin=10, rel=0.0)),
    # Materialize::kJ instances
    "cfg_poisson_mat": ("poisson", dict(W=24, H=20), dict(nl=3, lin=10, rel=0.0, materialize="j")),
    "cfg_arap_warp_mat": ("arap_warp", dict(W=24, H=20, nhandles=6), dict(nl=3, lin=10, rel=0.0, materialize="j")),
    "cfg_sfs_mat": ("sfs", dict(W=24, H=18), dict(nl=3, lin=10, rel=0.0, method="lm", materialize="j")),
    "cfg_arap_mesh_mat": ("arap_mesh", dict(n=8, nhandles=5), dict(nl=3, lin=10, rel=0.0, materialize="j")),
    "cfg_poisson_math": ("poisson", dict(W=24, H=20), dict(nl=3, lin=10, rel=0.0, materialize="jtj")),
    "cfg_arap_warp_math": ("arap_warp", dict(W=24, H=20, nhandles=6), dict(nl=3, lin=10, rel=0.0, materialize="jtj")),
    "cfg_arap_mesh_math": ("arap_mesh", dict(n=8, nhandles=5), dict(nl=3, lin=10, rel=0.0, materialize="jtj")),
}
