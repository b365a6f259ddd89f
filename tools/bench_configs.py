"""Full-size run of every BASELINE.json configuration on one B200.

Per config: host assembly time, device upload, matvec parity against the CPU
oracle (seeded U[-1,1] input, seed = config id), device-resident matvec
throughput with per-stage CUDA-event times and the near-field GEMM / M2L
roofline fractions, a GMRES solve (tol 1e-6, restart 50) and a capped-
iteration GMRES parity check against the oracle. cfg4 adds its 10-frequency
sweep (operator rebuilt per frequency), cfg5 its 64 Fibonacci plane waves
(batched matvec with nrhs = 64 and 64 GMRES solves).

    python tools/bench_configs.py [--configs 1,2,3,4,5] [--out profiles/r01_configs.jsonl]
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

# idle OpenMP workers of the oracle sleep instead of spinning, so they do not
# take host cores from the GPU solves timed after them (set before any load)
os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

HBM = 6541.8e9
FP64 = json.loads((ROOT / "profiles" / "r01_fp64_peak.json").read_text())["dmma_tflops"] * 1e12


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def pairs_of(data):
    m = data.counts
    return sum((m[0] - abs(int(o[0]))) * (m[1] - abs(int(o[1]))) * (m[2] - abs(int(o[2]))) for o in data.near_offsets)


def time_applies(op, x, steps):
    import torch

    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    op.set_stream(s.cuda_stream)
    for _ in range(3):
        op.matvec(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):
        op.matvec(x)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    op.enable_stage_timing(True)
    for _ in range(steps):
        op.matvec(x)
    st = op.stage_times()
    op.enable_stage_timing(False)
    return ms, {k: (v / max(1, st["applies"]) if k != "applies" else v) for k, v in st.items()}


def run_config(cid, args, out):
    import torch

    import oracle as O
    from paper_2201_12050_b200 import FmmOperators, Scene, gmres

    sc = Scene(cid, 0)
    rec = {"config": f"cfg{cid}", "lattice": list(sc.counts), "n_dof_cell": sc.n_dof, "N": sc.N,
           "k": sc.wavenumber}
    t = time.perf_counter()
    data = sc.assemble_fmm(4)
    rec["assembly_s"] = time.perf_counter() - t
    rec.update(near_offsets=data.n_near, far_offsets=data.n_far)
    nrhs = 64 if cid == 5 else 1
    t = time.perf_counter()
    op = FmmOperators(data, max_rhs=nrhs)
    rec["upload_s"] = time.perf_counter() - t
    path, lat, spec_bytes, mpb, sym_mask, sym_dev = op.near_path()
    rec["near_path"] = path
    rec["near_modes_per_block"] = mpb
    rec["near_symmetries"] = [g for g in range(1, 8) if sym_mask >> g & 1]
    rec["near_symmetry_deviation"] = sym_dev
    rec["near_lattice"] = list(lat)
    sizes, _ = op.spectrum()
    rec["fft_sizes"] = list(sizes)
    q = int(np.prod(sizes))

    rng = np.random.default_rng(cid)
    xh = rng.uniform(-1, 1, sc.N) + 1j * rng.uniform(-1, 1, sc.N)
    t = time.perf_counter()
    ora = O.OracleFmm(data)
    yo = ora.matvec(xh)
    rec["oracle_matvec_s"] = time.perf_counter() - t
    rec["oracle_threads"] = O.num_threads()
    rec["matvec_rel_err"] = rel(op.matvec(xh), yo)

    x = torch.from_numpy(xh).cuda()
    ms, st = time_applies(op, x, args.steps)
    pairs = pairs_of(data)
    flops = 8.0 * data.n_dof ** 2 * pairs
    rec["matvec_ms"] = ms
    rec["matvec_dof_per_s"] = sc.N / (ms * 1e-3)
    rec["stages_ms"] = st
    rec["near_gemm_tflops"] = flops / (st["near_gemm"] * 1e-3) / 1e12  # algorithmic (direct-path) flops
    rec["near_gemm_frac_of_fp64_peak"] = flops / (st["near_gemm"] * 1e-3) / FP64
    if path == "lattice":  # per-mode product streams the block spectrum
        qn = int(np.prod(lat))
        mb = spec_bytes + 2 * 16.0 * data.n_dof * qn  # stored blocks + x_hat read + y_hat written
        rec["near_mode_product_gb_per_s"] = mb / (st["near_mode_product"] * 1e-3) / 1e9
        rec["near_mode_product_frac_of_hbm"] = mb / (st["near_mode_product"] * 1e-3) / HBM
    lam_bytes = 16.0 * q * 625
    rec["m2l_lambda_gb_per_s"] = lam_bytes / (st["m2l"] * 1e-3) / 1e9
    rec["m2l_frac_of_hbm_lambda_only"] = lam_bytes / (st["m2l"] * 1e-3) / HBM
    k0 = op.kernel_launches()
    op.matvec(x)
    rec["kernel_launches_per_apply"] = op.kernel_launches() - k0
    out.write(json.dumps(rec) + "\n")
    out.flush()
    print(json.dumps(rec), flush=True)

    if nrhs > 1:
        # batched matvec over all 64 right-hand sides
        X = torch.from_numpy(np.concatenate([rng.uniform(-1, 1, sc.N) + 1j * rng.uniform(-1, 1, sc.N)
                                             for _ in range(nrhs)])).cuda()
        ms64, st64 = time_applies(op, X, max(2, args.steps // 10))
        r64 = {"config": f"cfg{cid}", "batched_nrhs": nrhs, "matvec_ms": ms64,
               "matvec_dof_per_s": nrhs * sc.N / (ms64 * 1e-3), "stages_ms": st64,
               "near_gemm_tflops": flops * nrhs / (st64["near_gemm"] * 1e-3) / 1e12}
        r64["near_gemm_frac_of_fp64_peak"] = r64["near_gemm_tflops"] * 1e12 / FP64
        y0 = op.matvec(X)[: sc.N].cpu().numpy()
        r64["batched_rel_err_rhs0_vs_oracle"] = rel(y0, ora.matvec(X[: sc.N].cpu().numpy()))
        out.write(json.dumps(r64) + "\n")
        print(json.dumps(r64), flush=True)

    # GMRES solve(s): cfg5's 64 plane waves in one lockstep batch
    solves = []
    t_all = time.perf_counter()
    if cid == 5:
        B = torch.from_numpy(np.concatenate([sc.rhs(f) for f in range(sc.n_rhs)])).cuda()
        gmres(op, B, tol=1e-6, restart=50, max_iter=2)  # warm: the handle's lockstep workspace (72 GB)
        torch.cuda.synchronize()
        t = time.perf_counter()
        reps = gmres(op, B, tol=1e-6, restart=50, max_iter=args.max_iter)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        for f, rep in enumerate(reps):
            solves.append({"field": f, "iterations": rep.iterations, "converged": rep.converged, "solve_s": dt,
                           "final_estimate": rep.residual_history[-1] if rep.residual_history else None})
    else:
        b = torch.from_numpy(sc.rhs(0)).cuda()
        gmres(op, b, tol=1e-6, restart=50, max_iter=2)  # warm: the handle's Krylov workspace
        torch.cuda.synchronize()
        t = time.perf_counter()
        rep = gmres(op, b, tol=1e-6, restart=50, max_iter=args.max_iter)
        torch.cuda.synchronize()
        solves.append({"field": 0, "iterations": rep.iterations, "converged": rep.converged,
                       "solve_s": time.perf_counter() - t,
                       "final_estimate": rep.residual_history[-1] if rep.residual_history else None})
    g = {"config": f"cfg{cid}", "gmres": "tol 1e-6 restart 50" + (" (64 RHS lockstep batch)" if cid == 5 else ""),
         "max_iter": args.max_iter, "solves": solves if len(solves) <= 4 else None,
         "n_solves": len(solves),
         # the solve calls only (cfg5: one lockstep batch); host RHS assembly and the warm-up excluded
         "total_solve_s": solves[0]["solve_s"] if cid == 5 else sum(s["solve_s"] for s in solves),
         "wall_incl_rhs_assembly_s": time.perf_counter() - t_all,
         "iterations_min_max": [min(s["iterations"] for s in solves), max(s["iterations"] for s in solves)],
         "all_converged": all(s["converged"] for s in solves)}
    # capped-iteration GMRES parity at full size (the oracle's full solve is hours on a CPU)
    cap = args.parity_iters
    b0 = sc.rhs(0)
    rep = gmres(op, b0, tol=1e-12, restart=50, max_iter=cap)
    t = time.perf_counter()
    xo, its, conv, hist = ora.gmres(b0, tol=1e-12, restart=50, max_iter=cap)
    g["parity_capped_iters"] = cap
    g["parity_oracle_s"] = time.perf_counter() - t
    g["parity_iterations"] = [rep.iterations, its]
    g["parity_solution_rel_err"] = rel(rep.solution, xo)
    g["parity_history_rel_err"] = rel(np.array(rep.residual_history), np.array(hist))
    out.write(json.dumps(g) + "\n")
    print(json.dumps(g), flush=True)

    if cid == 4 and args.sweep:
        op.close()
        for hz in sc.sweep_hz():
            sc.wavenumber = 2 * np.pi * hz / 343.0
            from paper_2201_12050_b200.fmm import assemble_far_gpu, assemble_near_gpu

            t = time.perf_counter()
            d = sc.assemble_fmm(4, skip_near_values=True, skip_far_values=True)  # offsets, U0, V0
            near = assemble_near_gpu(sc, d)
            far, _ = assemble_far_gpu(sc, d)
            torch.cuda.synchronize()
            ta = time.perf_counter() - t
            t = time.perf_counter()
            o = FmmOperators(d, near_blocks=near, far_blocks=far)
            tu = time.perf_counter() - t
            b = torch.from_numpy(sc.rhs(0)).cuda()
            torch.cuda.synchronize()
            t = time.perf_counter()
            rp = gmres(o, b, tol=1e-6, restart=50, max_iter=args.max_iter)
            torch.cuda.synchronize()
            r = {"config": "cfg4", "sweep_hz": hz, "assembly_s (offsets/U0/V0 on host, near blocks + K bank on GPU)": ta, "create_s": tu,
                 "solve_s": time.perf_counter() - t, "iterations": rp.iterations, "converged": rp.converged}
            out.write(json.dumps(r) + "\n")
            print(json.dumps(r), flush=True)
            o.close()
            del d, near, far


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--max-iter", type=int, default=1000)
    ap.add_argument("--parity-iters", type=int, default=8)
    ap.add_argument("--sweep", action="store_true")
    ap.add_argument("--out", default="gpurun_out/configs.jsonl")
    args = ap.parse_args()
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    with open(args.out, "a") as out:
        for c in args.configs.split(","):
            run_config(int(c), args, out)


if __name__ == "__main__":
    main()
