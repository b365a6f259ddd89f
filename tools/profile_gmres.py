"""Profiling driver: one GMRES solve (capped iterations) of a configuration."""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from tools.profile_matvec import Synthetic  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--restart", type=int, default=50)
    ap.add_argument("--nrhs", type=int, default=1)
    ap.add_argument("--dist", action="store_true", help="the slab-distributed CGS solver (one rank)")
    args = ap.parse_args()
    import torch

    from paper_2201_12050_b200 import FmmOperators, Scene, gmres
    from paper_2201_12050_b200.fmm import gmres_distributed

    if args.dist:
        gmres = gmres_distributed  # noqa: F811
    sc = Scene(args.config, 0)
    data = sc.assemble_fmm(4)
    op = FmmOperators(data, max_rhs=args.nrhs)
    b = torch.from_numpy(np.concatenate([sc.rhs(f % sc.n_rhs) for f in range(args.nrhs)])).cuda()
    gmres(op, b, tol=1e-12, restart=args.restart, max_iter=3)
    torch.cuda.synchronize()
    t = time.perf_counter()
    rep = gmres(op, b, tol=1e-12, restart=args.restart, max_iter=args.iters)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    its = rep.iterations if args.nrhs == 1 else max(r.iterations for r in rep)
    mv = torch.from_numpy(np.ones(data.N * args.nrhs, np.complex128)).cuda()
    op.matvec(mv)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10):
        op.matvec(mv)
    torch.cuda.synchronize()
    t_mv = (time.perf_counter() - t) / 10
    print(f"{'dist ' if args.dist else ''}{its} iterations in {dt * 1e3:.2f} ms = {dt / its * 1e3:.3f} ms/iteration "
          f"(nrhs {args.nrhs}); matvec {t_mv * 1e3:.3f} ms")


if __name__ == "__main__":
    main()
