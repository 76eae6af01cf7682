"""Strip sharding of grid plans across GPUs (the reference has
no multi-device path).

The plan's single grid domain is split into contiguous strips of axis-0 rows
(the slowest axis of the reference's row-major layout, problem.hpp:131-136).
A strip stores its owned rows plus `halo` rows on each side; the device
kernels keep global coordinates, so InBounds / index() / OOB reads behave as
in the unsharded problem.  Per PCG iteration the p halo is exchanged and the
p'Ap / r'z partials are gathered and summed in rank order, so every strip
takes the same alpha/beta.

Graph energies whose vertices are the domain's elements (the ARAP mesh) shard
as vertex ranges: the halo is the graph's row bandwidth (graph_halo_rows), a
strip keeps every edge touching its rows and counts only its own edges in
the cost.  `reorder=True` first renumbers the vertices by reverse
Cuthill-McKee (VertexOrder), so any mesh gets a small halo.

    # one process per GPU (torchrun), NCCL underneath:
    s = ShardedSolver(plan, global_data, rank, world, device)
    res = s.solve(); x = s.gather_x()
    # all strips on one GPU (tests, the single-device fake of SURVEY.md §4):
    g = LocalShardGroup(plan, global_data, world=3); res = g.solve(); x = g.gather_x()
"""
import ctypes
import threading
from dataclasses import dataclass
from typing import List

import numpy as np

from . import planinfo
from . import _lib
from ._lib import call
from .solver import CompiledPlan, EdgeTable, SolveData, Solver


def strip_rows(d0: int, world: int, rank: int):
    """Balanced contiguous partition of [0, d0) into `world` strips."""
    return (d0 * rank) // world, (d0 * (rank + 1)) // world


@dataclass
class Layout:
    d0: int              # axis-0 extent of the grid domain
    S: int               # elements per axis-0 row
    unknown_ch: List[int]
    array_ch: List[int]
    halo: int


def graph_halo_rows(graphs, S: int) -> int:
    """Row bandwidth of the bound graphs (max row distance between two vertices
    of one edge, vertex v in row v // S): the halo a strip needs so that it
    stores every endpoint of the edges touching its rows."""
    h = 0
    for g in graphs:
        v = np.asarray(g.verts, np.int64).reshape(-1, g.arity) // S
        if v.size:
            h = max(h, int((v.max(axis=1) - v.min(axis=1)).max()))
    return h


def layout(plan: CompiledPlan, data: SolveData = None) -> Layout:
    info = planinfo.parse(plan.text)
    dims = dict(info.dims)
    dims.update(plan.dims)
    names = list(info.dims.keys())

    def shape(dd):
        return [dims[names[i]] for i in dd]

    doms = [tuple(f[2]) for f in info.fields["U"] + info.fields["A"] + info.fields["C"]]
    if not doms or len(set(doms)) != 1:
        raise ValueError("strip sharding needs every field on one grid domain")
    shp = shape(doms[0])
    h = ctypes.c_int()
    call("mo_plan_halo_rows", plan._h, ctypes.byref(h))
    S = int(np.prod(shp[1:])) if len(shp) > 1 else 1
    halo = h.value
    if data is not None and data.graphs:
        halo = max(halo, graph_halo_rows(data.graphs, S))
    return Layout(shp[0], S, [f[1] for f in info.fields["U"]], [f[1] for f in info.fields["A"]], halo)


def _rows_of(vec, d0, row_elems, lo, hi):
    return vec.reshape(d0, row_elems)[lo:hi].reshape(-1)


def local_data(plan: CompiledPlan, data: SolveData, row0: int, row1: int) -> SolveData:
    """The strip's SolveData: rows [lo, hi) of every field (halos included).
    Graphs stay global: the session keeps the edges touching its rows."""
    L = layout(plan, data)
    lo, hi = max(0, row0 - L.halo), min(L.d0, row1 + L.halo)
    x, off, parts = np.asarray(data.x), 0, []
    for C in L.unknown_ch:
        n = L.d0 * L.S * C
        parts.append(_rows_of(x[off:off + n], L.d0, L.S * C, lo, hi))
        off += n
    arrays = [_rows_of(np.asarray(a), L.d0, L.S * C, lo, hi) for a, C in zip(data.arrays, L.array_ch)]
    return SolveData(x=np.concatenate(parts) if parts else x[:0], arrays=arrays, params=list(data.params),
                     graphs=[EdgeTable(g.arity, g.verts) for g in data.graphs])


def owned_x(plan: CompiledPlan, xloc: np.ndarray, row0: int, row1: int, halo: int = None) -> List[np.ndarray]:
    """Per unknown field, the strip's owned rows of its local x."""
    L = layout(plan)
    if halo is not None:
        L.halo = halo
    lo, hi = max(0, row0 - L.halo), min(L.d0, row1 + L.halo)
    out, off = [], 0
    for C in L.unknown_ch:
        n = (hi - lo) * L.S * C
        out.append(xloc[off:off + n].reshape(hi - lo, L.S * C)[row0 - lo:row1 - lo].reshape(-1))
        off += n
    return out


def assemble_x(plan: CompiledPlan, owned: List[List[np.ndarray]]) -> np.ndarray:
    """Global x (reference column layout) from every strip's owned rows (rank order)."""
    L = layout(plan)
    return np.concatenate([np.concatenate([o[f] for o in owned]) for f in range(len(L.unknown_ch))])


class VertexOrder:
    """Reverse Cuthill-McKee renumbering of a graph energy's vertex domain, so
    that vertex strips need only a small halo (the renumbered bandwidth) on
    any mesh, not just banded ones.  Valid when the domain is 1-D and no grid
    program reads it at a nonzero offset (per-vertex terms only, like the ARAP
    mesh's fit): then the energy is invariant under the permutation."""

    def __init__(self, plan: CompiledPlan, data: SolveData):
        from scipy.sparse import coo_matrix
        from scipy.sparse.csgraph import reverse_cuthill_mckee
        L = layout(plan)
        if L.S != 1 or L.halo != 0:
            raise ValueError("vertex renumbering needs a 1-D domain read at offset 0 only")
        n = L.d0
        rows, cols = [], []
        for g in data.graphs:
            v = np.asarray(g.verts, np.int64).reshape(-1, g.arity)
            for a in range(g.arity):
                for b in range(g.arity):
                    if a != b:
                        rows.append(v[:, a])
                        cols.append(v[:, b])
        r = np.concatenate(rows) if rows else np.zeros(0, np.int64)
        c = np.concatenate(cols) if cols else np.zeros(0, np.int64)
        adj = coo_matrix((np.ones(r.size, np.int8), (r, c)), shape=(n, n)).tocsr()
        self.perm = np.asarray(reverse_cuthill_mckee(adj, symmetric_mode=True), np.int64)  # new -> old
        self.inv = np.empty(n, np.int64)
        self.inv[self.perm] = np.arange(n)  # old -> new
        self.L = L

    def apply(self, data: SolveData) -> SolveData:
        """The same problem with vertex i renamed inv[i]."""
        L, n = self.L, self.L.d0
        x, off, parts = np.asarray(data.x), 0, []
        for C in L.unknown_ch:
            parts.append(x[off:off + n * C].reshape(n, C)[self.perm].reshape(-1))
            off += n * C
        arrays = [np.asarray(a).reshape(n, C)[self.perm].reshape(-1) for a, C in zip(data.arrays, L.array_ch)]
        graphs = [EdgeTable(g.arity, self.inv[np.asarray(g.verts, np.int64)].astype(np.uint64)) for g in data.graphs]
        return SolveData(x=np.concatenate(parts) if parts else x[:0], arrays=arrays, params=list(data.params),
                         graphs=graphs)

    def restore_x(self, xp: np.ndarray) -> np.ndarray:
        """x in the caller's vertex numbering from the renumbered x."""
        L, n, off, parts = self.L, self.L.d0, 0, []
        for C in L.unknown_ch:
            f = np.empty((n, C), xp.dtype)
            f[self.perm] = xp[off:off + n * C].reshape(n, C)
            parts.append(f.reshape(-1))
            off += n * C
        return np.concatenate(parts) if parts else xp[:0]


class LocalShardGroup:
    """`world` strip sessions of one plan on one GPU, driven from one host
    thread each (the LocalComm transport): the single-device fake that tests
    the exact partition / halo / reduction schedule the NCCL path runs."""

    def __init__(self, plan: CompiledPlan, data: SolveData, world: int, device: int = 0, reorder: bool = False):
        self.plan, self.world = plan, world
        self.order = VertexOrder(plan, data) if reorder else None
        if self.order:
            data = self.order.apply(data)
        L = layout(plan, data)
        self.halo = L.halo
        self._w = ctypes.c_void_p()
        call("mo_world_create_local", int(world), int(device), ctypes.byref(self._w))
        self.comms, self.rows = [], []
        for r in range(world):
            c = ctypes.c_void_p()
            call("mo_comm_create_local", self._w, r, ctypes.byref(c))
            self.comms.append(c)
            self.rows.append(strip_rows(L.d0, world, r))
        # Construction refreshes (collective halo exchanges): one thread per strip.
        self.solvers = list(range(world))
        self.solvers = self._parallel(
            lambda r: Solver(plan, local_data(plan, data, *self.rows[r]), device, comm=self.comms[r], rows=self.rows[r],
                             halo=self.halo))

    def _parallel(self, fn):
        out, err = [None] * self.world, []

        def run(r):
            try:
                out[r] = fn(self.solvers[r])  # (ints during construction)
            except Exception as e:  # pragma: no cover - surfaced below
                err.append(e)

        ts = [threading.Thread(target=run, args=(r,)) for r in range(self.world)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        if err:
            raise err[0]
        return out

    def solve(self):
        return self._parallel(lambda s: s.solve())

    def cost(self):
        return self._parallel(lambda s: s.cost())

    def gather_x(self):
        x = assemble_x(self.plan, [owned_x(self.plan, s.get_x(), *rw, halo=self.halo)
                                   for s, rw in zip(self.solvers, self.rows)])
        return self.order.restore_x(x) if self.order else x

    def close(self):
        for s in self.solvers:
            s.__del__()
        self.solvers = []
        for c in self.comms:
            _lib.lib.mo_comm_destroy(c)
        self.comms = []
        if self._w:
            _lib.lib.mo_world_destroy(self._w)
            self._w = None

    def __del__(self):
        if getattr(self, "_w", None):
            self.close()


class ShardedSolver:
    """One strip per process (torchrun, one GPU per rank): the NCCL unique id
    is broadcast with torch.distributed, halos and partials then travel over
    NCCL on the session's stream."""

    def __init__(self, plan: CompiledPlan, data: SolveData, rank: int, world: int, device: int,
                 reorder: bool = False):
        import torch.distributed as dist
        self.plan, self.rank, self.world = plan, rank, world
        self.order = VertexOrder(plan, data) if reorder else None  # deterministic: same on every rank
        if self.order:
            data = self.order.apply(data)
        L = layout(plan, data)
        self.halo = L.halo
        uid = (ctypes.c_char * 128)()
        if rank == 0:
            call("mo_nccl_unique_id", uid, 128)
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=0)
        uid = (ctypes.c_char * 128).from_buffer_copy(box[0])
        self._c = ctypes.c_void_p()
        call("mo_comm_create_nccl", uid, 128, rank, world, device, ctypes.byref(self._c))
        self.rows = strip_rows(L.d0, world, rank)
        self.solver = Solver(plan, local_data(plan, data, *self.rows), device, comm=self._c, rows=self.rows,
                             halo=self.halo)

    def solve(self):
        return self.solver.solve()

    def gather_x(self):
        import torch.distributed as dist
        mine = owned_x(self.plan, self.solver.get_x(), *self.rows, halo=self.halo)
        allp = [None] * self.world
        dist.all_gather_object(allp, mine)
        x = assemble_x(self.plan, allp)
        return self.order.restore_x(x) if self.order else x
