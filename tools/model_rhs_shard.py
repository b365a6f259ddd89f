"""cfg5 (64 right-hand sides) sharded over P GPUs: every
rank holds the full operator and solves 64/P right-hand sides as one lockstep
batch, with no collective inside the solves. On one GPU this times exactly what
one rank of P does — the batched product and a lockstep GMRES step at 64/P
right-hand sides — so the P-GPU efficiency is measured per rank, not modelled
(only the final gather of the reports is left out: a few hundred bytes).

    python tools/model_rhs_shard.py [--config 5] [--iters 10]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--rhs", type=int, default=64)
    ap.add_argument("--ranks", default="1,2,4,8")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--steps", type=int, default=5)
    args = ap.parse_args()
    import torch

    from bench import workload
    from paper_2201_12050_b200 import FmmOperators, gmres
    from paper_2201_12050_b200.fmm import assemble_near_gpu

    sc, desc = workload(args.config)
    data = sc.assemble_fmm(4, skip_near_values=True)
    near = assemble_near_gpu(sc, data, device=0)
    op = FmmOperators(data, device=0, near_blocks=near, max_rhs=args.rhs)
    rng = np.random.default_rng(args.config)
    out = {"config": args.config, "workload": desc, "rhs_total": args.rhs, "P": {}}
    for P in [int(v) for v in args.ranks.split(",")]:
        k = args.rhs // P
        x = torch.from_numpy(rng.uniform(-1, 1, data.N * k) + 1j * rng.uniform(-1, 1, data.N * k)).cuda()
        for _ in range(2):
            op.matvec(x)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(args.steps):
            op.matvec(x)
        torch.cuda.synchronize()
        mv = (time.perf_counter() - t) / args.steps
        b = torch.from_numpy(np.concatenate([sc.rhs(f % sc.n_rhs) for f in range(k)])).cuda()
        gmres(op, b, tol=1e-30, restart=50, max_iter=2)
        torch.cuda.synchronize()
        solve = {}
        for its in (args.iters, 2 * args.iters):  # steady-state step = difference of two solve lengths
            t = time.perf_counter()
            gmres(op, b, tol=1e-30, restart=50, max_iter=its)
            torch.cuda.synchronize()
            solve[its] = time.perf_counter() - t
        step = (solve[2 * args.iters] - solve[args.iters]) / args.iters
        out["P"][P] = {"rhs_per_rank": k, "batched_product_ms": 1e3 * mv, "lockstep_step_ms": 1e3 * step,
                       "note": f"step = (solve of {2 * args.iters} its - solve of {args.iters} its) / {args.iters}, "
                               f"Krylov steps j = {args.iters}..{2 * args.iters - 1} of a restart-50 cycle"}
        print(json.dumps({"P": P, **out["P"][P]}), flush=True)
    base = out["P"][min(out["P"])]
    for P, v in out["P"].items():
        v["product_efficiency"] = base["batched_product_ms"] / (P * v["batched_product_ms"]) * min(out["P"])
        v["solve_efficiency"] = base["lockstep_step_ms"] / (P * v["lockstep_step_ms"]) * min(out["P"])
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
