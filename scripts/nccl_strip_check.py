"""Multi-rank strip check (one GPU per rank, torchrun): the same grid solved
unsharded on rank 0 and in `world` axis-0 strips over NCCL (halo send/recv,
fixed-order all-gathers, CUDA-graph captured stages); the trajectories must
agree (only dot-product summation order differs).  Exit 0 and print
`NCCL_STRIPS_OK` on rank 0 when they do.

    python -m torch.distributed.run --standalone --nproc-per-node 2 scripts/nccl_strip_check.py [poisson|arap_warp]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1604_06525_b200 import Method, Precision, SolveConfig, Solver, load_plan, workloads  # noqa: E402
from paper_1604_06525_b200.sharded import ShardedSolver  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    name = sys.argv[1] if len(sys.argv) > 1 else "poisson"
    prob = workloads.poisson(96, 64) if name == "poisson" else workloads.arap_warp(96, 64, nhandles=8)
    c = SolveConfig(method=Method.kGaussNewton, precision=Precision.kF64, nonlinear_iters=3, linear_iters=10,
                    pcg_rel_tol=0.0)
    sh = ShardedSolver(load_plan(prob.name, c, prob.dims), prob.data(np.float64), rank, world, local)
    r = sh.solve()
    x = sh.gather_x()
    ok = True
    if rank == 0:
        ref_data = prob.data(np.float64)
        ref = Solver(load_plan(prob.name, c, prob.dims), ref_data, device=local).solve()
        for a, b in zip(r.trace, ref.trace):
            ok &= abs(a.cost - b.cost) <= 1e-9 * abs(b.cost) and a.pcg_iters == b.pcg_iters
        ok &= bool(np.allclose(x, ref_data.x, rtol=1e-8, atol=1e-8))
        print("NCCL_STRIPS_OK" if ok else f"NCCL_STRIPS_MISMATCH {[t.cost for t in r.trace]} {[t.cost for t in ref.trace]}",
              flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
