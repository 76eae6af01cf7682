"""Reference-API behaviour on the GPU with hand-derived expectations
(reference proj/tests/test_solver.cpp): callbacks, bind errors, graph scatter
values, single precision, iteration caps."""
import numpy as np
import pytest

from helpers import Golden
from paper_1604_06525_b200 import (EdgeTable, Method, MoError, Precision, SolveConfig, SolveData, Solver,
                                   StopReason)
from paper_1604_06525_b200.solver import CompiledPlan

pytestmark = pytest.mark.gpu


def plan_of(golden_name, **cfg):
    g = Golden(golden_name)
    c = SolveConfig(**cfg) if cfg else g.cfg
    with open(f"{__import__('helpers').GOLDEN}/{golden_name}.moplan") as f:
        return CompiledPlan(f.read(), c)


def test_chain_hand_values():
    """test_solver.cpp:39-77."""
    s = Solver(plan_of("chain"), SolveData(x=np.zeros(2), arrays=[np.array([1.0, 0.0])]))
    assert s.num_cols() == 2 and s.num_rows() == 4
    assert s.cost() == 1.0
    np.testing.assert_array_equal(s.residuals(), [-1.0, 0.0, 0.0, 0.0])
    s.build_normal()
    np.testing.assert_array_equal(s.rhs(), [2.0, 0.0])
    np.testing.assert_array_equal(s.precond(), [4.0, 4.0])
    np.testing.assert_array_equal(s.apply_jtj([1.0, 0.0]), [4.0, -2.0])


def test_chain_one_gn_step():
    """test_solver.cpp:79-101."""
    data = SolveData(x=np.zeros(2), arrays=[np.array([1.0, 0.0])])
    s = Solver(plan_of("chain", nonlinear_iters=1), data)
    r = s.solve()
    assert data.x[0] == pytest.approx(2 / 3, rel=1e-12)
    assert data.x[1] == pytest.approx(1 / 3, rel=1e-12)
    assert r.final_cost == pytest.approx(1 / 3, rel=1e-12)
    assert r.reason == StopReason.kIterLimit
    assert len(r.trace) == 1 and r.trace[0].accepted and r.trace[0].radius == 0.0
    assert r.trace[0].pcg_iters <= 2 and r.unconstrained == 0 and not r.nonfinite_kernels
    assert r.trace_csv().startswith("iter,cost,accepted,radius,pcg_iters,wall_ms")


def test_graph_scatter_values():
    """test_solver.cpp:155-186."""
    data = SolveData(x=np.array([3.0, 1.0]), graphs=[EdgeTable(2, np.array([0, 1], np.uint64))])
    s = Solver(plan_of("graph"), data)
    assert s.num_rows() == 1 and s.cost() == 4.0
    s.build_normal()
    np.testing.assert_array_equal(s.rhs(), [-4.0, 4.0])
    np.testing.assert_array_equal(s.precond(), [2.0, 2.0])
    np.testing.assert_array_equal(s.apply_jtj([1.0, 0.0]), [2.0, -2.0])
    assert s.solve().unconstrained == 0
    assert s.cost() == pytest.approx(0.0, abs=1e-20)


def test_callback_mutates_arrays():
    """test_solver.cpp:409-430."""
    data = SolveData(x=np.zeros(2), arrays=[np.array([1.0, 2.0])])
    p = plan_of("chain", nonlinear_iters=2)
    calls = []

    def cb(it, d):
        calls.append(it)
        if it == 0:
            d.arrays[0] = np.array([5.0, 6.0])

    s = Solver(p, data)
    s.solve(cb)
    assert calls == [0, 1]
    # chain energy: (x0-a0)^2 + (x1-a1)^2 + (x0-x1)^2 -> least squares solution
    A = np.array([[1, 0], [0, 1], [1, -1]], float)
    sol = np.linalg.lstsq(A, np.array([5.0, 6.0, 0.0]), rcond=None)[0]
    np.testing.assert_allclose(data.x, sol, rtol=1e-10)


def test_callback_grows_graph():
    """test_solver.cpp:432-453."""
    text = open(f"{__import__('helpers').GOLDEN}/graph.moplan").read()
    from paper_1604_06525_b200 import plan as mkplan
    p = mkplan(text, SolveConfig(nonlinear_iters=2), dims={"N": 3})
    # energy P(a) - P(b): consistent system; grow from one edge to two
    data = SolveData(x=np.array([1.0, 0.0, 0.0]), graphs=[EdgeTable(2, np.array([0, 1], np.uint64))])
    s = Solver(p, data)
    assert s.num_rows() == 1

    def cb(it, d):
        if it == 0:
            d.graphs[0] = EdgeTable(2, np.array([0, 1, 1, 2], np.uint64))

    r = s.solve(cb)
    assert s.num_rows() == 2
    assert data.x[0] - data.x[1] == pytest.approx(0.0, abs=1e-10)
    assert data.x[1] - data.x[2] == pytest.approx(0.0, abs=1e-10)
    assert r.final_cost == pytest.approx(0.0, abs=1e-18)


def test_single_precision_chain():
    """test_solver.cpp:488-507."""
    data = SolveData(x=np.zeros(2, np.float32), arrays=[np.array([1.0, 0.0], np.float32)])
    s = Solver(plan_of("chain", precision=Precision.kF32, nonlinear_iters=1), data)
    assert s.cost() == 1.0
    s.build_normal()
    assert s.rhs()[0] == np.float32(2.0) and s.precond()[0] == np.float32(4.0)
    r = s.solve()
    assert data.x.dtype == np.float32
    assert data.x[0] == pytest.approx(2 / 3, rel=1e-6)
    assert r.final_cost == pytest.approx(1 / 3, rel=1e-6)


def test_bind_errors():
    """test_solver.cpp:509-537."""
    p = plan_of("chain")
    with pytest.raises(MoError) as e:
        Solver(p, SolveData(x=np.zeros(1), arrays=[np.array([1.0, 0.0])]))
    assert e.value.code == "BindError"
    with pytest.raises(MoError) as e:
        Solver(p, SolveData(x=np.zeros(2), arrays=[np.array([1.0])]))
    assert e.value.code == "BindError"
    gp = plan_of("graph")
    with pytest.raises(MoError) as e:
        Solver(gp, SolveData(x=np.zeros(2)))
    assert e.value.code == "BindError"
    with pytest.raises(MoError) as e:
        Solver(gp, SolveData(x=np.zeros(2), graphs=[EdgeTable(3, np.array([0, 1, 1], np.uint64))]))
    assert e.value.code == "BindError"


def test_vertex_out_of_range_rejected():
    """test_exec.cpp:302-322: validated before any write."""
    gp = plan_of("graph")
    with pytest.raises(MoError) as e:
        s = Solver(gp, SolveData(x=np.zeros(2), graphs=[EdgeTable(2, np.array([0, 5], np.uint64))]))
        s.cost()
    assert e.value.code == "IndexOutOfRange"


def test_iteration_cap_truncates():
    """test_pcg.cpp:176-195 via the solver: linear_iters caps PCG iterations."""
    g = Golden("cfg_poisson_f64")
    c = g.cfg
    c.linear_iters = 1
    c.nonlinear_iters = 1
    data = g.data()
    s = Solver(load_plan_cfg(g, c), data)
    r = s.solve()
    assert r.trace[0].pcg_iters == 1 and not r.indefinite_operator


def load_plan_cfg(g, c):
    from paper_1604_06525_b200 import load_plan
    return load_plan(f"{__import__('helpers').GOLDEN}/{g.name}.moplan", c)


def test_lm_radius_triples_on_quadratic():
    """test_solver.cpp:298-321."""
    data = SolveData(x=np.zeros(2), arrays=[np.array([1.0, 0.0])])
    s = Solver(plan_of("chain", method=Method.kLevenbergMarquardt, nonlinear_iters=2), data)
    r = s.solve()
    assert r.trace[0].accepted and r.trace[0].radius == 1e4
    assert r.trace[1].radius == pytest.approx(3e4, rel=1e-10)
    prev = 1.0
    for row in r.trace:
        if row.accepted:
            assert row.cost < prev
            prev = row.cost


@pytest.mark.parametrize("first,second", [("quarter", "none"), ("none", "quarter"), ("quarter", "half")])
def test_rebound_masks_rebuild_the_active_lists(first, second):
    """The Poisson apply walks a list of active tiles and the PCG vector
    kernels a list of active column groups, both built with the masks
    (mo_session.cu build_tile_lists / build_group_list).  Re-binding the mask
    array between solves (nothing excluded <-> a quarter or half active) must
    give exactly what a fresh solver on the new data gives."""
    from paper_1604_06525_b200 import Method, Precision, SolveConfig, load_plan, workloads
    prob = workloads.poisson(96, 64)
    W, H = prob.dims["W"], prob.dims["H"]
    i = np.arange(W)[:, None]
    j = np.arange(H)[None, :]

    def mask(kind):
        if kind == "none":
            return np.zeros(W * H)
        keep = (i >= W // 4) & (i < 3 * W // 4) & (j >= H // 4) & (j < 3 * H // 4)
        if kind == "half":
            keep = np.broadcast_to(i < W // 2, (W, H))
        return np.where(keep, 0.0, 1.0).reshape(-1)

    cfg = SolveConfig(method=Method.kGaussNewton, precision=Precision.kF64, nonlinear_iters=2, linear_iters=8,
                      pcg_rel_tol=0.0)
    plan = load_plan(prob.name, cfg, prob.dims)
    d = prob.data(np.float64)
    d.arrays[1] = mask(first)
    s = Solver(plan, d)
    s.solve()
    d.x[:] = prob.data(np.float64).x
    d.arrays[1] = mask(second)
    s._bind_all()
    s.refresh()
    r = s.solve()
    fresh = prob.data(np.float64)
    fresh.arrays[1] = mask(second)
    r2 = Solver(load_plan(prob.name, cfg, prob.dims), fresh).solve()
    assert [t.pcg_iters for t in r.trace] == [t.pcg_iters for t in r2.trace]
    np.testing.assert_allclose(d.x, fresh.x, rtol=1e-12, atol=1e-12 * np.max(np.abs(fresh.x)))
    assert abs(r.final_cost - r2.final_cost) <= 1e-12 * abs(r2.final_cost)
