"""Seeded synthetic inputs for the five BASELINE.json configs.

Every random draw comes from a counter-based splitmix64 stream so the same
values can be regenerated anywhere (numpy here, the reference driver reads the
arrays we hand it).  Values are produced in float64 and rounded once to the
session precision, so the CPU reference and the GPU see identical inputs.

    prob = poisson(512, 512)              # config 1
    prob = arap_warp(1024, 1024)          # config 2
    prob = sfs(640, 480)                  # config 3 (LM)
    prob = arap_mesh(448)                 # config 4 (200,704 vertices)
    prob = poisson(8192, 8192) / arap_warp(8192, 8192)   # config 5
"""
from dataclasses import dataclass, field
from typing import Dict, List

import numpy as np

from .solver import EdgeTable, SolveData


def uniform(seed: int, n: int) -> np.ndarray:
    """U[0,1) float64 from splitmix64(seed * 2^32 + i)."""
    i = np.arange(n, dtype=np.uint64) + np.uint64((seed & 0xFFFFFFFF) << 32)
    with np.errstate(over="ignore"):
        z = i * np.uint64(0x9E3779B97F4A7C15) + np.uint64(0x632BE59BD9B4E019)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def normal(seed: int, n: int) -> np.ndarray:
    """N(0,1) via Box-Muller on two splitmix64 streams."""
    u1 = uniform(seed, n)
    u2 = uniform(seed + 7919, n)
    return np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * np.pi * u2)


@dataclass
class Problem:
    name: str            # plan name under paper_1604_06525_b200/plans
    dims: Dict[str, int]
    x: np.ndarray
    arrays: List[np.ndarray]
    params: List[float]
    graphs: List[EdgeTable] = field(default_factory=list)
    method: str = "gn"   # gn | lm
    energy: str = ""     # energy file stem (for the reference driver)

    def data(self, dtype) -> SolveData:
        return SolveData(x=self.x.astype(dtype), arrays=[a.astype(dtype) for a in self.arrays],
                         params=list(self.params),
                         graphs=[EdgeTable(g.arity, g.verts.copy()) for g in self.graphs])

    def bytes_per(self, dtype) -> int:
        s = np.dtype(dtype).itemsize
        return self.x.size * s + sum(a.size * s for a in self.arrays)


def poisson(W: int = 512, H: int = 512) -> Problem:
    """Poisson image editing float3 (Fig. 27).  T ~ U[0,1)^3 (seed 1), X0 ~
    U[0,1)^3 (seed 2); M = 0 inside the centred rectangle [W/4,3W/4)x[H/4,3H/4)."""
    n = W * H
    T = uniform(1, 3 * n)
    X0 = uniform(2, 3 * n)
    i = np.arange(W)[:, None]
    j = np.arange(H)[None, :]
    inside = (i >= W // 4) & (i < 3 * W // 4) & (j >= H // 4) & (j < 3 * H // 4)
    M = np.where(inside, 0.0, 1.0).reshape(-1)
    return Problem("poisson", {"W": W, "H": H}, X0, [T, M], [], energy="poisson")


def _handles(seed: int, count: int, extent: int) -> np.ndarray:
    return np.minimum((uniform(seed, count) * extent).astype(np.int64), extent - 1)


def arap_warp(W: int = 1024, H: int = 1024, nhandles: int = 64) -> Problem:
    """ARAP image warping (Fig. 24).  Ur = (i, j); Off0 = Ur; Ang0 = 0; M = 0;
    C = -1 except `nhandles` seeded pixels with C = Ur + U[0,5)^2;
    w_fit = 10, w_reg = 1."""
    n = W * H
    i, j = np.meshgrid(np.arange(W, dtype=np.float64), np.arange(H, dtype=np.float64), indexing="ij")
    Ur = np.stack([i.reshape(-1), j.reshape(-1)], axis=1)
    C = -np.ones((n, 2))
    hi = _handles(11, nhandles, W)
    hj = _handles(12, nhandles, H)
    hp = hi * H + hj
    C[hp] = Ur[hp] + 5.0 * uniform(13, 2 * nhandles).reshape(nhandles, 2)
    x = np.concatenate([Ur.reshape(-1), np.zeros(n)])
    M = np.zeros(n)
    return Problem("arap_warp", {"W": W, "H": H}, x, [Ur.reshape(-1), C.reshape(-1), M], [10.0, 1.0],
                   energy="arap_warp")


def sfs(W: int = 640, H: int = 480) -> Problem:
    """Shape from shading (Fig. 26), LM.  D = 1 + 0.1 sin(0.02 i) cos(0.03 j);
    X0 = D + N(0, 0.002^2) (seed 1); Im = 0.5 + 0.3 sin(0.05 i + 0.04 j);
    f = 525, u = (W/2, H/2), SH lighting L1..L9 fixed."""
    i, j = np.meshgrid(np.arange(W, dtype=np.float64), np.arange(H, dtype=np.float64), indexing="ij")
    D = (1.0 + 0.1 * np.sin(0.02 * i) * np.cos(0.03 * j)).reshape(-1)
    X0 = D + 0.002 * normal(1, W * H)
    Im = (0.5 + 0.3 * np.sin(0.05 * i + 0.04 * j)).reshape(-1)
    L = [0.5, 0.1, -0.3, 0.2, 0.05, 0.01, -0.02, 0.03, 0.01]
    params = [1.0, 0.5, 0.2, 525.0, 525.0, W / 2.0, H / 2.0] + L
    return Problem("sfs", {"W": W, "H": H}, X0, [D, Im], params, method="lm", energy="sfs")


def grid_mesh_edges(n: int, rows: int = 0) -> np.ndarray:
    """Both directions of every edge of a rows x n grid mesh (rows = n by
    default), vertex-major order."""
    rows = rows or n
    v = np.arange(rows * n, dtype=np.uint64).reshape(rows, n)
    right = np.stack([v[:, :-1], v[:, 1:]], axis=-1)
    down = np.stack([v[:-1, :], v[1:, :]], axis=-1)
    e = []
    for a in (right, down):
        a = a.reshape(-1, 2)
        e.append(np.stack([a, a[:, ::-1]], axis=1).reshape(-1, 2))
    return np.concatenate(e).reshape(-1)


def arap_mesh(n: int = 448, nhandles: int = 64, rows: int = 0) -> Problem:
    """ARAP mesh deformation (Fig. 25) on a rows x n grid mesh (rows = n by
    default; n=448 gives 200,704 vertices and 801,024 directed edges).
    Ur = (r, c, 0); Off0 = Ur; Ang0 = 0; C = -1e6 except handles
    C = Ur + U[0,3)^3; w_fit = 10, w_reg = 1."""
    rows = rows or n
    N = rows * n
    r, c = np.meshgrid(np.arange(rows, dtype=np.float64), np.arange(n, dtype=np.float64), indexing="ij")
    Ur = np.stack([r.reshape(-1), c.reshape(-1), np.zeros(N)], axis=1)
    C = np.full((N, 3), -1e6)
    h = _handles(21, nhandles, N)
    C[h] = Ur[h] + 3.0 * uniform(22, 3 * nhandles).reshape(nhandles, 3)
    x = np.concatenate([Ur.reshape(-1), np.zeros(3 * N)])
    g = EdgeTable(2, grid_mesh_edges(n, rows))
    return Problem("arap_mesh", {"N": N}, x, [Ur.reshape(-1), C.reshape(-1)], [10.0, 1.0], [g],
                   energy="arap_mesh")


CONFIGS = {
    "poisson": poisson,
    "arap_warp": arap_warp,
    "sfs": sfs,
    "arap_mesh": arap_mesh,
}
