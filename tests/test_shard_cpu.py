"""Host-side logic of the multi-GPU strip path on CPU with torch.distributed
(gloo, world_size 2, 127.0.0.1): strip partition, local slicing with halos,
halo consistency between neighbours, and the all-gather that reassembles the
global unknown vector — the same Python the NCCL ranks run."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1604_06525_b200 import load_plan, workloads
from paper_1604_06525_b200.sharded import assemble_x, layout, local_data, owned_x, strip_rows


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, dims, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        prob = workloads.CONFIGS[name](**dims)
        plan = load_plan(prob.name, dims=prob.dims)
        data = prob.data(np.float64)
        L = layout(plan, data)
        rows = strip_rows(L.d0, world, rank)
        loc = local_data(plan, data, *rows)
        # halo rows of x must equal the neighbour's owned rows
        mine = owned_x(plan, loc.x, *rows, halo=L.halo)
        allp = [None] * world
        dist.all_gather_object(allp, {"rows": rows, "x": loc.x, "owned": mine})
        lo = max(0, rows[0] - L.halo)
        ok = True
        off = 0
        for f, C in enumerate(L.unknown_ch):
            n = (min(L.d0, rows[1] + L.halo) - lo) * L.S * C
            block = loc.x[off:off + n].reshape(-1, L.S * C)
            off += n
            gx = assemble_x(plan, [a["owned"] for a in allp])
            goff = sum(L.d0 * L.S * c for c in L.unknown_ch[:f])
            gfield = gx[goff:goff + L.d0 * L.S * C].reshape(L.d0, L.S * C)
            ok &= np.array_equal(block, gfield[lo:lo + block.shape[0]])
        x = assemble_x(plan, [a["owned"] for a in allp])
        q.put((rank, bool(ok), bool(np.array_equal(x, data.x)), rows, L.halo))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,dims", [("poisson", dict(W=20, H=12)), ("arap_warp", dict(W=18, H=10)),
                                       ("arap_mesh", dict(n=9, nhandles=4))])
def test_gloo_world2_partition_halo_gather(name, dims):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, name, dims, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert [r[0] for r in res] == [0, 1]
    assert all(r[1] for r in res), "halo rows differ from the neighbour's owned rows"
    assert all(r[2] for r in res), "all-gathered owned rows do not reassemble x"
    (r0, r1), (s0, s1) = res[0][3], res[1][3]
    assert r0 == 0 and r1 == s0 and s1 == dims.get("W", dims.get("n", 0) ** 2)
    assert res[0][4] >= 1


def test_strip_rows_cover_and_balance():
    for d0 in (7, 64, 8192):
        for world in (1, 2, 3, 8):
            rows = [strip_rows(d0, world, r) for r in range(world)]
            assert rows[0][0] == 0 and rows[-1][1] == d0
            assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
            sizes = [b - a for a, b in rows]
            assert max(sizes) - min(sizes) <= 1


def test_graph_halo_is_the_row_bandwidth():
    from paper_1604_06525_b200 import EdgeTable
    from paper_1604_06525_b200.sharded import graph_halo_rows
    prob = workloads.arap_mesh(9, nhandles=4)  # 9x9 grid mesh, vertex = r * 9 + c
    assert graph_halo_rows(prob.graphs, 1) == 9
    assert graph_halo_rows([EdgeTable(3, np.array([0, 5, 2, 7, 7, 7], np.uint64))], 2) == 2
    plan = load_plan(prob.name, dims=prob.dims)
    assert layout(plan, prob.data(np.float64)).halo == 9


def test_rcm_renumbering_shrinks_the_halo_and_round_trips():
    """A mesh with scrambled vertex ids has a bandwidth ~N; reverse
    Cuthill-McKee brings it back to ~the grid width, and restore_x undoes the
    renumbering exactly."""
    from paper_1604_06525_b200.sharded import VertexOrder, graph_halo_rows
    prob = workloads.arap_mesh(12, nhandles=5)
    n = 144
    rng = np.random.default_rng(3)
    p = rng.permutation(n)  # scramble: old vertex i -> p[i]
    data = prob.data(np.float64)
    inv = np.argsort(p)
    x = data.x.reshape(2, n, 3)[:, inv].reshape(-1)  # new id j holds old vertex inv[j]
    arrays = [a.reshape(n, 3)[inv].reshape(-1) for a in data.arrays]
    from paper_1604_06525_b200 import EdgeTable, SolveData
    graphs = [EdgeTable(2, p[np.asarray(g.verts, np.int64)].astype(np.uint64)) for g in data.graphs]
    scrambled = SolveData(x=x, arrays=arrays, params=data.params, graphs=graphs)
    assert graph_halo_rows(scrambled.graphs, 1) > 60
    plan = load_plan(prob.name, dims=prob.dims)
    vo = VertexOrder(plan, scrambled)
    ordered = vo.apply(scrambled)
    assert graph_halo_rows(ordered.graphs, 1) <= 24
    np.testing.assert_array_equal(vo.restore_x(ordered.x), scrambled.x)
