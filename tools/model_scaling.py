"""Per-rank timing of the slab-distributed product and GMRES on ONE GPU, and
the multi-GPU model built from it.

For P = 1, 2, 4, 8 and every rank r of P, the operator gets a slab plan over a
simulated communicator (fpbem_cu_comm_simulated: rank r of P alone on this
device; its exchanges move only its own blocks and count the bytes the real
NCCL exchange would send). The rank's whole share of a product — P2M, the DFTs
below the slab axis on its planes, pack, own-block copy, the DFTs along the
slab axis, its near-field block products and Λ on its columns, unpack, the
inverse DFTs, L2P — is timed with CUDA events on the handle's stream. Nothing
waits on another rank, so this is the compute side of a P-GPU product exactly;
the exchanges are modelled from the counted bytes:

    t_P = max_r t_r + n_exchanges x (latency + max_r bytes_r / bandwidth)

with the NVLink-5 all-to-all figures stated in the output (an assumption: no
multi-GPU box was available). Efficiency = t_1 / (P t_P), t_1 the single-GPU
product (the regular apply, not the slab path).

Run on a GPU box: python tools/model_scaling.py --config 3 [--steps 50]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

# NVLink 5 / NVSwitch all-to-all assumption (per GPU, per direction): 900 GB/s
# link rate; NCCL's measured all-to-all bus bandwidth on 8 x B200 is lower for
# MB-sized messages, so the model uses a conservative effective rate plus a
# fixed cost per grouped send/recv exchange
A2A_GBS = 450.0
A2A_LAT_US = 15.0
AR_LAT_US = 12.0  # a small all-reduce (GMRES scalars)


def timed(fn, steps, stream):
    import torch

    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(3):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / steps)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--ranks", default="1,2,4,8")
    ap.add_argument("--gmres-iters", type=int, default=40)
    ap.add_argument("--only", default="", help="P,r: time only rank r of P (e.g. under ncu)")
    ap.add_argument("--no-gmres", action="store_true")
    args = ap.parse_args()

    import torch

    from paper_2201_12050_b200 import FmmOperators
    from paper_2201_12050_b200.fmm import SimulatedCommunicator, assemble_near_gpu, gmres_distributed
    from bench import workload

    sc, desc = workload(args.config)
    data = sc.assemble_fmm(4, skip_near_values=True)
    near = assemble_near_gpu(sc, data, device=0)
    op = FmmOperators(data, device=0, near_blocks=near, near_path="lattice")
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    op.set_stream(stream.cuda_stream)
    rng = np.random.default_rng(args.config)
    xh = rng.uniform(-1, 1, data.N) + 1j * rng.uniform(-1, 1, data.N)
    x = torch.from_numpy(xh).cuda()
    t1 = timed(lambda: op.matvec(x), args.steps, stream)
    print(json.dumps({"config": args.config, "workload": desc, "single_gpu_apply_ms": t1}), flush=True)
    b = torch.from_numpy(sc.rhs(0)).cuda()

    out = {"config": args.config, "workload": desc, "t1_ms": t1, "a2a_GBps": A2A_GBS, "a2a_latency_us": A2A_LAT_US,
           "allreduce_latency_us": AR_LAT_US, "P": {}}
    only = tuple(int(v) for v in args.only.split(",")) if args.only else None
    for P in ([only[0]] if only else [int(v) for v in args.ranks.split(",")]):
        per = []
        for r in ([only[1]] if only else range(P)):
            comm = SimulatedCommunicator(0, P, r)
            op.set_slabs(comm)
            lo, hi = op.slab_rows()
            xs = x[lo:hi].contiguous()
            comm.traffic(reset=True)
            op.matvec_slab(xs)
            torch.cuda.synchronize()
            sent, n_coll = comm.traffic(reset=True)
            t = timed(lambda: op.matvec_slab(xs), args.steps, stream)
            # GMRES on the slabs: a fixed number of inner steps (no restart), per step
            comm.traffic(reset=True)
            gs, g_sent, g_coll, its = 0.0, 0, 0, 1
            if not args.no_gmres:
                # warm call first (workspace allocation), then the timed one
                # (a simulated rank's solve runs on its partial operator: its control flow is
                # for timing only, and a run that ends early is simply not timed)
                try:
                    gmres_distributed(op, b, tol=1e-30, restart=4, max_iter=4)
                    torch.cuda.synchronize()
                    comm.traffic(reset=True)
                    t0 = time.perf_counter()
                    rep = gmres_distributed(op, b, tol=1e-30, restart=args.gmres_iters, max_iter=args.gmres_iters)
                    torch.cuda.synchronize()
                    gs = time.perf_counter() - t0
                    g_sent, g_coll = comm.traffic(reset=True)
                    its = max(1, rep.iterations)
                except RuntimeError as e:
                    print(json.dumps({"P": P, "rank": r, "gmres_not_timed": str(e)}), flush=True)
            per.append({"rank": r, "rows": hi - lo, "apply_ms": t, "a2a_bytes": sent, "exchanges": n_coll,
                        "gmres_ms_per_iter": 1e3 * gs / its, "gmres_iters": its,
                        "gmres_bytes_per_iter": g_sent / its, "gmres_collectives_per_iter": g_coll / its})
            print(json.dumps({"P": P, **per[-1]}), flush=True)
            op.set_slabs(None)
            comm.close()
        tmax = max(p["apply_ms"] for p in per)
        bmax = max(p["a2a_bytes"] for p in per)
        nex = per[0]["exchanges"]
        comm_ms = 0.0 if P == 1 else nex * (A2A_LAT_US * 1e-3 + bmax / (A2A_GBS * 1e9) * 1e3)
        tP = tmax + comm_ms
        # GMRES step: slab product + the Gram-Schmidt all-reduces (latency-bound)
        g_compute = max(p["gmres_ms_per_iter"] for p in per)
        g_coll = per[0]["gmres_collectives_per_iter"]
        g_comm = 0.0 if P == 1 else comm_ms + max(0.0, g_coll - nex) * AR_LAT_US * 1e-3
        out["P"][P] = {"max_rank_apply_ms": tmax, "min_rank_apply_ms": min(p["apply_ms"] for p in per),
                       "a2a_bytes_max_rank": bmax, "exchanges_per_apply": nex, "modeled_comm_ms": comm_ms,
                       "modeled_apply_ms": tP, "modeled_efficiency_vs_single_gpu": t1 / (P * tP),
                       "gmres_max_rank_ms_per_iter": g_compute, "gmres_collectives_per_iter": g_coll,
                       "modeled_gmres_ms_per_iter": g_compute + g_comm, "ranks": per}
        print(json.dumps({"P": P, "summary": {k: v for k, v in out["P"][P].items() if k != "ranks"}}), flush=True)
    print(json.dumps(out), flush=True)
    op.close()


if __name__ == "__main__":
    main()
