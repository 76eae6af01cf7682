"""Pin the C restatement (oracle/mo_oracle.c) against the unmodified
reference's golden outputs: it must reproduce them BIT FOR BIT (same
sequential order, same libm, no contraction) before it may serve as the
checker for GPU parity tests at sizes the goldens do not cover."""
import numpy as np
import pytest

from helpers import Golden, golden_names
from oracle.cref import Oracle, OracleError


def bits_equal(a, b):
    a = np.atleast_1d(np.asarray(a))
    b = np.atleast_1d(np.asarray(b, dtype=a.dtype))
    return a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))


ERR_RC = {"IndexOutOfRange": 11, "BindError": 15, "InternalError": 18}


@pytest.mark.parametrize("name", golden_names())
def test_oracle_reproduces_reference_bitwise(name):
    g = Golden(name)
    err = g.ref("error")
    if err is None:
        run_oracle(g, name)
        return
    # the reference threw: the restatement raises the same Err code
    with pytest.raises(OracleError) as ei:
        run_oracle(g, name)
    assert ei.value.rc == ERR_RC[bytes(err).decode().split(":")[0]], str(ei.value)


def run_oracle(g, name):
    plan_text = open(f"{__import__('helpers').GOLDEN}/{name}.moplan").read()
    o = Oracle(plan_text, f64=g.prec == "f64", cfg=g.cfg)
    data = g.data()
    o.bind(data)
    assert o.num_cols() == int(g.ref("num_cols")[0])
    assert o.num_rows() == int(g.ref("num_rows")[0])
    assert bits_equal(o.excluded(), g.ref("excluded"))
    for cmd in g.cmds:
        if cmd == "cost":
            assert bits_equal(np.float64(o.cost()), g.ref("cost")[0])
        elif cmd == "residuals":
            assert bits_equal(o.residuals(), g.ref("residuals"))
        elif cmd == "normal":
            b, m = o.build_normal()
            assert bits_equal(b, g.ref("b")) and bits_equal(m, g.ref("m"))
        elif cmd == "linearize":
            offs, col, val = o.linearize()
            assert bits_equal(offs, g.ref("j_offs")) and bits_equal(col, g.ref("j_col"))
            assert bits_equal(val, g.ref("j_val"))
            if g.ref("h_offs") is not None:
                ho, hc, hv = o.normal_matrix()
                assert bits_equal(ho, g.ref("h_offs")) and bits_equal(hc, g.ref("h_col"))
                assert bits_equal(hv, g.ref("h_val"))
        elif cmd == "jtj":
            assert bits_equal(o.apply_jtj(g.z["v"].astype(g.dtype)), g.ref("jtj"))
        elif cmd == "solve":
            r, tr = o.solve()
            assert r.reason == int(g.ref("reason")[0])
            assert bits_equal(np.float64(r.final_cost), g.ref("final_cost")[0])
            assert list(tr["accepted"]) == list(g.ref("trace_accepted"))
            assert list(tr["pcg"]) == list(g.ref("trace_pcg"))
            assert bits_equal(tr["cost"], g.ref("trace_cost"))
            assert bits_equal(tr["radius"], g.ref("trace_radius"))
            assert r.unconstrained == int(g.ref("unconstrained")[0])
            assert r.nonfinite_kernels == int(g.ref("nonfinite_kernels")[0])
            assert r.indefinite == int(g.ref("indefinite")[0])
            assert bits_equal(o.get_x(), g.ref("x_final"))


def test_oracle_bind_errors_mirror_reference():
    g = Golden("chain")
    plan_text = open(f"{__import__('helpers').GOLDEN}/chain.moplan").read()
    o = Oracle(plan_text)
    d = g.data()
    d.x = np.zeros(1)
    with pytest.raises(Exception) as e:
        o.bind(d)
    assert e.value.rc == 15  # 1 + Err::kBindError
