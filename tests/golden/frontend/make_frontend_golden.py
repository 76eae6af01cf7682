"""Reference verdicts on malformed / unusual energy sources, for
tests/test_frontend.py: each source is planned by the UNMODIFIED reference
(oracle/_ref/ref_driver: compile_source + plan) and the Err name it raises
(or "ok") is stored in errors.json.  Run here (needs /root/reference)."""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", ".."))
from oracle import pyoracle  # noqa: E402
from paper_1604_06525_b200.solver import SolveData  # noqa: E402

H = "dim W 4\ndim H 3\nparam p\nunknown X [W, H] : 2\narray A [W, H]\ngraph G (a, b)\n"
SOURCES = {
    "syntax_trailing_op": "dim W 2\nunknown X [W]\nenergy X(0) +\n",
    "syntax_bad_char": "dim W 2\nunknown X [W]\nenergy X(0) $ 1\n",
    "syntax_unknown_stmt": "dim W 2\nfield X [W]\n",
    "syntax_reserved_name": "dim W 2\nunknown sin [W]\n",
    "syntax_redeclared": "dim W 2\nunknown X [W]\narray X [W]\n",
    "syntax_dim_extent": "dim W 2.5\n",
    "undeclared_field": "dim W 2\nunknown X [W]\nenergy Y(0)\n",
    "undeclared_dim": "unknown X [W]\n",
    "arity_offsets": "dim W 2\nunknown X [W]\nenergy X(0, 1)\n",
    "arity_param_access": H + "energy p(0)\n",
    "arity_builtin": H + "energy sin(X(0,0)[0], 1)\n",
    "nonconst_offset": H + "energy X(p, 0)[0]\n",
    "nonconst_exponent": H + "energy pow(X(0,0)[0], p)\n",
    "mixed_graph_stencil": H + "dim N 4\nunknown Q [N]\nenergy Q(G.a) - X(0,0)[0]\n",
    "domain_no_fields": H + "energy p * 2\n",
    "nonboolean_select": H + "energy select(X(0,0)[0], 1, 0)\n",
    "nonboolean_exclude": H + "exclude A(0,0)\n",
    "shape_width": H + "energy X(0,0) + vec(1, 2, 3)\n",
    "index_channel": H + "energy X(0,0)[2]\n",
    "index_slice": H + "energy slice(X(0,0), 1, 3)\n",
    "cyclic_computed": H + "computed S freeze = S(0,0) + A(0,0)\n",
    "graph_slot_in_computed": H + "dim N 4\nunknown Q [N]\ncomputed S freeze = Q(G.a)\n",
    "graph_inbounds": H + "dim N 4\nunknown Q [N]\nenergy select(inbounds(1), Q(G.a), 0)\n",
    "ok_rotate_normalize": H + "energy normalize(rotate2d(A(0,0), X(0,0) - X(1,0)))\n",
    "ok_pow_fraction": H + "energy pow(abs(X(0,0)[0]) + 1, 2.5) + pow(X(0,1)[1] * X(0,1)[1] + 1, -0.5)\n",
    "ok_dot_slice_vec": H + "energy dot(X(0,0), vec(A(0,0), 1)) - slice(vec(X(-1,0), A(0,0)), 1, 2)\n",
    "ok_comments": "# header\ndim W 3 # trailing\nunknown X [W]\nenergy X(0) - 1.5e-1 # done\n",
}


def main():
    d = SolveData(x=np.zeros(2), arrays=[], params=[], graphs=[])
    out = {}
    for name, src in SOURCES.items():
        r = pyoracle.run_ref(src, d, [])
        err = r.get("error")
        code = bytes(err).decode().split(":")[0] if err is not None else "ok"
        # (the zero-size data never binds: a BindError means compile + plan passed)
        out[name] = {"source": src, "reference": "ok" if code == "BindError" else code}
    with open(os.path.join(HERE, "errors.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    for k, v in out.items():
        print(f"{k:28s} {v['reference']}")


if __name__ == "__main__":
    main()
