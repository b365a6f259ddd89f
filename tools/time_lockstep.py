"""Lockstep (64-RHS) GMRES step cost along a restart cycle: warm solves capped at
k iterations for several k; the per-step cost is the slope between them."""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    from bench import workload
    from paper_2201_12050_b200 import FmmOperators, gmres
    from paper_2201_12050_b200.fmm import assemble_near_gpu

    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    sc, desc = workload(cfg)
    data = sc.assemble_fmm(4, skip_near_values=True)
    near = assemble_near_gpu(sc, data, device=0)
    op = FmmOperators(data, device=0, near_blocks=near, max_rhs=nrhs)
    if "--torch-stream" in sys.argv:  # the handle on a torch stream, as bench.py / bench_configs.py set it
        st = torch.cuda.Stream()
        torch.cuda.set_stream(st)
        op.set_stream(st.cuda_stream)
    if "--oracle" in sys.argv:  # the CPU oracle's OpenMP product first, as bench_configs.py's parity check
        import os

        os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")
        import oracle as O

        O.OracleFmm(sc.assemble_fmm(4)).matvec(np.ones(data.N, dtype=np.complex128))
    if "--host-apply" in sys.argv:  # one host-pointer product first, as bench_configs.py's parity check
        op.matvec(np.ones(data.N, dtype=np.complex128))
    if "--host-data" in sys.argv:  # the operator from the host-assembled blocks, as bench_configs.py
        op.close()
        op = FmmOperators(sc.assemble_fmm(4), device=0, max_rhs=nrhs)
    if "--timed-applies" in sys.argv:  # stage timing on and off first, as bench_configs.py does
        X = torch.zeros(data.N * nrhs, dtype=torch.complex128, device="cuda")
        op.enable_stage_timing(True)
        op.matvec(X)
        op.stage_times()
        op.enable_stage_timing(False)
    B = torch.from_numpy(np.concatenate([sc.rhs(f % sc.n_rhs) for f in range(nrhs)])).cuda()
    gmres(op, B, tol=1e-6, restart=50, max_iter=2)
    torch.cuda.synchronize()
    prev = (0, 0.0)
    for k in (20, 80):
        t = time.perf_counter()
        reps = gmres(op, B, tol=1e-6, restart=50, max_iter=k)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        its = max(r.iterations for r in reps)
        print(json.dumps({"cfg": cfg, "nrhs": nrhs, "max_iter": k, "solve_s": dt, "max_its": its,
                          "ms_per_step_since_prev": 1e3 * (dt - prev[1]) / max(1, k - prev[0])}), flush=True)
        prev = (k, dt)


if __name__ == "__main__":
    main()
