"""One-off check: the simulated-communicator slab product and slab GMRES stay finite (rank 0 of 2, cfg3)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    from bench import workload
    from paper_2201_12050_b200 import FmmOperators
    from paper_2201_12050_b200.fmm import SimulatedCommunicator, assemble_near_gpu, gmres_distributed

    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    sc, _ = workload(cfg)
    data = sc.assemble_fmm(4, skip_near_values=True)
    near = assemble_near_gpu(sc, data, device=0)
    op = FmmOperators(data, device=0, near_blocks=near, near_path="lattice")
    x = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, data.N) + 0j).cuda()
    b = torch.from_numpy(sc.rhs(0)).cuda()
    for P, r in [(1, 0), (2, 0), (2, 1), (4, 3)]:
        comm = SimulatedCommunicator(0, P, r)
        op.set_slabs(comm)
        lo, hi = op.slab_rows()
        for k in range(3):
            y = op.matvec_slab(x[lo:hi].contiguous())
            print(P, r, k, "finite", bool(torch.isfinite(y).all()), float(y.abs().max()), flush=True)
        try:
            rep = gmres_distributed(op, b, tol=1e-30, restart=4, max_iter=4)
            print(P, r, "gmres ok", rep.iterations, rep.residual_history, flush=True)
        except RuntimeError as e:
            print(P, r, "gmres failed:", e, flush=True)
        op.set_slabs(None)
        comm.close()


if __name__ == "__main__":
    main()
