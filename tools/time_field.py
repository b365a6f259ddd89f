"""Time field evaluation (postproc::evaluate_field): the device kernel over a
grid of observation points vs the host restatement on a bounded sample of the
same points (all host threads), per config. Usage: python tools/time_field.py [cfg ...]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2201_12050_b200 import Scene  # noqa: E402
from paper_2201_12050_b200.fmm import evaluate_field_gpu  # noqa: E402
from paper_2201_12050_b200.host import grid_points  # noqa: E402


def main():
    cfgs = [int(c) for c in sys.argv[1:]] or [1, 2, 3, 4]
    for cid in cfgs:
        sc = Scene(cid, 0)
        c = sc.cell()
        lo = np.min(c["centroid"], axis=0)
        hi = np.max(c["centroid"], axis=0) + np.asarray(sc.pitch) * (np.asarray(sc.counts) - 1)
        pts = grid_points(lo - 1.0, hi + 1.0, (8, 8, 4))  # 256 points around the array
        sol = np.random.default_rng(cid).uniform(-1, 1, sc.N) + 1j * np.random.default_rng(cid + 1).uniform(-1, 1, sc.N)
        p_inc = sc.incident(pts)
        sol_d = torch.from_numpy(sol).cuda()
        pinc_d = torch.from_numpy(p_inc).cuda()
        evaluate_field_gpu(sc, sol_d, pts[:4], p_incident=pinc_d[:4])  # warm-up
        torch.cuda.synchronize()
        t = time.perf_counter()
        dev = evaluate_field_gpu(sc, sol_d, pts, p_incident=pinc_d)
        torch.cuda.synchronize()
        t_dev = time.perf_counter() - t
        n_s = 2 if sc.N > 200_000 else 8  # bounded host sample
        t = time.perf_counter()
        host = sc.field_host(sol, pts[:n_s])
        t_host = time.perf_counter() - t
        err = float(np.linalg.norm(dev.cpu().numpy()[:n_s] - host) / np.linalg.norm(host))
        evals = len(pts) * sc.N
        print(json.dumps({"config": cid, "N": sc.N, "points": len(pts), "device_s": round(t_dev, 4),
                          "device_Gelem_per_s": round(evals / t_dev / 1e9, 3),
                          "host_sample_points": n_s, "host_s_per_point": round(t_host / n_s, 4),
                          "host_threads": os.cpu_count(), "speedup_per_point": round(t_host / n_s / (t_dev / len(pts)), 1),
                          "rel_err_vs_host": err}), flush=True)


if __name__ == "__main__":
    main()
