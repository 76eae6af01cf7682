"""Strip sharding on one GPU (the single-device multi-strip fake of SURVEY.md
§4/§8e): N strip sessions exchange halos and gather partials through the
LocalComm transport, running exactly the schedule the NCCL path runs.  The
sharded solve must reproduce the unsharded one (fixed PCG iterations); only
the summation order of the dot products differs."""
import numpy as np
import pytest

from paper_1604_06525_b200 import Method, Precision, SolveConfig, Solver, load_plan, workloads
from paper_1604_06525_b200.sharded import LocalShardGroup

pytestmark = pytest.mark.gpu

CASES = {
    "poisson": (lambda: workloads.poisson(40, 24), "gn"),
    "arap_warp": (lambda: workloads.arap_warp(48, 20, nhandles=6), "gn"),
    "sfs": (lambda: workloads.sfs(36, 20), "lm"),
    # graph energy: vertex strips, halo = the mesh's row bandwidth (§8f rank 3)
    "arap_mesh": (lambda: workloads.arap_mesh(12, nhandles=5), "gn"),
    "arap_mesh_lm": (lambda: workloads.arap_mesh(12, nhandles=5, rows=17), "lm"),
}


def cfg(method, prec):
    return SolveConfig(method=Method.kLevenbergMarquardt if method == "lm" else Method.kGaussNewton,
                       precision=Precision.kF64 if prec == "f64" else Precision.kF32,
                       nonlinear_iters=3, linear_iters=8, pcg_rel_tol=0.0)


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", list(CASES))
def test_strips_match_unsharded(name, world, prec):
    make, method = CASES[name]
    prob = make()
    dt = np.float64 if prec == "f64" else np.float32
    c = cfg(method, prec)
    ref_data = prob.data(dt)
    ref = Solver(load_plan(prob.name, c, prob.dims), ref_data).solve()

    g = LocalShardGroup(load_plan(prob.name, c, prob.dims), prob.data(dt), world)
    try:
        results = g.solve()
        x = g.gather_x()
    finally:
        g.close()
    tol = 1e-9 if prec == "f64" else 2e-4
    for r in results:  # every strip takes the same steps
        assert [t.accepted for t in r.trace] == [t.accepted for t in ref.trace]
        assert [t.pcg_iters for t in r.trace] == [t.pcg_iters for t in ref.trace]
        for a, b in zip(r.trace, ref.trace):
            assert abs(a.cost - b.cost) <= tol * abs(b.cost), (a.cost, b.cost)
        assert abs(r.final_cost - ref.final_cost) <= tol * abs(ref.final_cost)
        assert r.unconstrained == ref.unconstrained
    scale = np.max(np.abs(ref_data.x))
    np.testing.assert_allclose(x, ref_data.x, rtol=tol * 10, atol=tol * 10 * scale)


@pytest.mark.parametrize("variant", ["gather", "twophase", "stream", "tma", "warp", "gprog", "tma4", "ws", "lc",
                                     "lct"])
def test_overlapped_strip_apply_every_variant(variant, monkeypatch):
    """Grid strips apply the interior rows while the p halo is exchanged on a
    side stream, then the border rows (mo_session.cu apply_overlapped): each
    J^T J p variant over three row ranges must give the unsharded solve, and
    MO_B200_NO_OVERLAP (exchange first, one launch) the same steps."""
    monkeypatch.setenv("MO_B200_JTJ", variant)
    prob = workloads.arap_warp(60, 20, nhandles=6)
    c = cfg("gn", "f64")
    ref_data = prob.data(np.float64)
    ref = Solver(load_plan(prob.name, c, prob.dims), ref_data).solve()
    xs = {}
    for overlap in (True, False):
        if overlap:
            monkeypatch.delenv("MO_B200_NO_OVERLAP", raising=False)
        else:
            monkeypatch.setenv("MO_B200_NO_OVERLAP", "1")
        g = LocalShardGroup(load_plan(prob.name, c, prob.dims), prob.data(np.float64), 3)
        try:
            results = g.solve()
            xs[overlap] = g.gather_x()
        finally:
            g.close()
        for r in results:
            assert [t.pcg_iters for t in r.trace] == [t.pcg_iters for t in ref.trace]
            assert abs(r.final_cost - ref.final_cost) <= 1e-9 * abs(ref.final_cost)
    scale = np.max(np.abs(ref_data.x))
    for x in xs.values():
        np.testing.assert_allclose(x, ref_data.x, rtol=1e-8, atol=1e-8 * scale)


@pytest.mark.parametrize("name", ["poisson", "sfs", "arap_mesh"])
def test_peer_reductions_bitwise_equal_allgather(name, monkeypatch):
    """The one-shot peer-memory reductions (k_peer_fin: slots in every rank's
    exchange block, release/acquire flags, rank-order sum) give bitwise the
    same solve as the all-gather + k_global_fin path (MO_B200_NO_P2P=1).
    The single-GPU transport takes the peer path on request only
    (MO_B200_LOCAL_P2P=1, mo_comm.cpp)."""
    monkeypatch.setenv("MO_B200_LOCAL_P2P", "1")
    make, method = CASES[name]
    prob = make()
    c = cfg(method, "f64")
    out = {}
    for p2p in (True, False):
        if p2p:
            monkeypatch.delenv("MO_B200_NO_P2P", raising=False)
        else:
            monkeypatch.setenv("MO_B200_NO_P2P", "1")
        g = LocalShardGroup(load_plan(prob.name, c, prob.dims), prob.data(np.float64), 3)
        try:
            g.solve()  # (the peer path starts with a session's second solve)
            res = g.solve()
            out[p2p] = (g.gather_x(), [[t.cost for t in r.trace] for r in res])
        finally:
            g.close()
    np.testing.assert_array_equal(out[True][0], out[False][0])
    assert out[True][1] == out[False][1]


@pytest.mark.parametrize("name", ["poisson", "arap_mesh"])
def test_nccl_transport_world1(name, monkeypatch):
    """The NCCL transport (dlopen'ed libnccl, unique id via torch.distributed,
    all-gather on the session stream) on the one GPU available: world 1.
    (The unsharded reference solve walks the column mask like a strip does,
    MO_B200_NO_GROUP_LIST=1, so the comparison is bitwise.)"""
    monkeypatch.setenv("MO_B200_NO_GROUP_LIST", "1")
    import os
    import socket

    import torch.distributed as dist

    from paper_1604_06525_b200.sharded import ShardedSolver
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        prob = workloads.poisson(32, 16) if name == "poisson" else workloads.arap_mesh(10, nhandles=4)
        c = cfg("gn", "f64")
        ref_data = prob.data(np.float64)
        ref = Solver(load_plan(prob.name, c, prob.dims), ref_data).solve()
        sh = ShardedSolver(load_plan(prob.name, c, prob.dims), prob.data(np.float64), 0, 1, 0)
        r = sh.solve()
        x = sh.gather_x()
        if name == "poisson":  # same kernels and reduction order: bitwise
            assert [t.cost for t in r.trace] == [t.cost for t in ref.trace]
            np.testing.assert_array_equal(x, ref_data.x)
        else:  # the strip path gathers graphs unfused (other p'Ap partials)
            for a, b in zip(r.trace, ref.trace):
                assert abs(a.cost - b.cost) <= 1e-9 * abs(b.cost)
            np.testing.assert_allclose(x, ref_data.x, rtol=1e-8, atol=1e-8)
    finally:
        dist.destroy_process_group()


def test_single_strip_equals_unsharded_bitwise(monkeypatch):
    """world=1: the shard path with no neighbours is the unsharded algorithm
    (with the unsharded PCG walking the column mask like a strip,
    MO_B200_NO_GROUP_LIST=1)."""
    monkeypatch.setenv("MO_B200_NO_GROUP_LIST", "1")
    prob = workloads.poisson(32, 16)
    c = cfg("gn", "f64")
    ref_data = prob.data(np.float64)
    ref = Solver(load_plan(prob.name, c, prob.dims), ref_data).solve()
    g = LocalShardGroup(load_plan(prob.name, c, prob.dims), prob.data(np.float64), 1)
    try:
        r = g.solve()[0]
        x = g.gather_x()
    finally:
        g.close()
    assert [t.cost for t in r.trace] == [t.cost for t in ref.trace]
    np.testing.assert_array_equal(x, ref_data.x)


@pytest.mark.parametrize("world", [2, 4])
def test_scrambled_mesh_strips_with_rcm(world):
    """Any vertex numbering: the strips renumber by reverse Cuthill-McKee
    (halo = the renumbered bandwidth) and still reproduce the unsharded solve
    of the caller's numbering."""
    from paper_1604_06525_b200 import EdgeTable, SolveData
    prob = workloads.arap_mesh(16, nhandles=6)
    n = 256
    p = np.random.default_rng(7).permutation(n)
    inv = np.argsort(p)
    d = prob.data(np.float64)
    data = SolveData(x=d.x.reshape(2, n, 3)[:, inv].reshape(-1), arrays=[a.reshape(n, 3)[inv].reshape(-1) for a in d.arrays],
                     params=d.params, graphs=[EdgeTable(2, p[np.asarray(g.verts, np.int64)].astype(np.uint64))
                                              for g in d.graphs])
    c = cfg("gn", "f64")
    ref_data = SolveData(x=data.x.copy(), arrays=data.arrays, params=data.params, graphs=data.graphs)
    ref = Solver(load_plan(prob.name, c, prob.dims), ref_data).solve()
    g = LocalShardGroup(load_plan(prob.name, c, prob.dims), data, world, reorder=True)
    try:
        assert g.halo < 40
        results = g.solve()
        x = g.gather_x()
    finally:
        g.close()
    for r in results:
        for a, b in zip(r.trace, ref.trace):
            assert abs(a.cost - b.cost) <= 1e-9 * abs(b.cost), (a.cost, b.cost)
    np.testing.assert_allclose(x, ref_data.x, rtol=1e-8, atol=1e-8)


@pytest.mark.parametrize("name", ["poisson", "arap_warp"])
def test_nccl_two_ranks(name):
    """Two processes, one GPU each, strips over NCCL (halo send/recv and the
    fixed-order all-gathers inside captured stage graphs) against the
    unsharded solve; runs whenever two GPUs are visible."""
    import subprocess
    import sys

    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (this box has one)")
    root = __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--standalone", "--nproc-per-node", "2",
                        "scripts/nccl_strip_check.py", name], cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "NCCL_STRIPS_OK" in r.stdout, (r.stdout[-2000:], r.stderr[-2000:])
