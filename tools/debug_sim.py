"""One-off check: the simulated-communicator slab product and slab GMRES stay finite and take the
expected time (cfg3), with the handle on torch's stream as bench.py / model_scaling.py set it."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    from bench import workload
    from paper_2201_12050_b200 import FmmOperators
    from paper_2201_12050_b200.fmm import SimulatedCommunicator, assemble_near_gpu, gmres_distributed

    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    use_stream = "--stream" in sys.argv
    sc, _ = workload(cfg)
    data = sc.assemble_fmm(4, skip_near_values=True)
    near = assemble_near_gpu(sc, data, device=0)
    op = FmmOperators(data, device=0, near_blocks=near, near_path="lattice")
    if use_stream:
        st = torch.cuda.Stream()
        torch.cuda.set_stream(st)
        op.set_stream(st.cuda_stream)
    x = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, data.N) + 0j).cuda()
    b = torch.from_numpy(sc.rhs(0)).cuda()
    for P, r in [(0, 0), (1, 0), (2, 0), (4, 3)]:
        comm = SimulatedCommunicator(0, P, r) if P else None
        op.set_slabs(comm)
        lo, hi = op.slab_rows()
        for k in range(20):
            y = op.matvec_slab(x[lo:hi].contiguous())
        print(P, r, "finite", bool(torch.isfinite(y).all()), float(y.abs().max()), flush=True)
        for its in (4, 40):
            try:
                torch.cuda.synchronize()
                t = time.perf_counter()
                rep = gmres_distributed(op, b, tol=1e-30, restart=its, max_iter=its)
                torch.cuda.synchronize()
                dt = time.perf_counter() - t
                print(P, r, its, "gmres ok", rep.iterations, f"{1e3 * dt / rep.iterations:.3f} ms/it",
                      rep.residual_history[-1], flush=True)
            except RuntimeError as e:
                print(P, r, its, "gmres failed:", e, flush=True)
        op.set_slabs(None)
        if comm:
            comm.close()


if __name__ == "__main__":
    main()
