"""Time the K-bank assembly per frequency: host TranslationTable loop
(Scene.assemble_fmm, all host threads) vs the device bank (fpbem_cu_m2l_bank)
and the spectrum build from it. Usage: python tools/time_far_bank.py [cfg ...]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2201_12050_b200 import FmmOperators, Scene  # noqa: E402
from paper_2201_12050_b200.fmm import assemble_far_gpu  # noqa: E402


def main():
    cfgs = [int(c) for c in sys.argv[1:]] or [3, 4, 5, 2]
    for cid in cfgs:
        sc = Scene(cid, 0)
        sc.assemble_fmm(4, skip_near_values=True, skip_far_values=True)  # warm the host tables
        t = time.perf_counter()
        d_host = sc.assemble_fmm(4, skip_near_values=True)
        t_host_full = time.perf_counter() - t
        t = time.perf_counter()
        d = sc.assemble_fmm(4, skip_near_values=True, skip_far_values=True)
        t_host_shape = time.perf_counter() - t
        far, _ = assemble_far_gpu(sc, d)  # warm-up (term tables uploaded once per process)
        torch.cuda.synchronize()
        reps = 5
        t = time.perf_counter()
        for _ in range(reps):
            far, _ = assemble_far_gpu(sc, d)
        torch.cuda.synchronize()
        t_dev = (time.perf_counter() - t) / reps
        err = float(np.linalg.norm(far.cpu().numpy() - np.asarray(d_host.far_blocks)) /
                    np.linalg.norm(np.asarray(d_host.far_blocks)))
        print(json.dumps({"config": cid, "n_far": d.n_far, "host_bank_s": round(t_host_full - t_host_shape, 4),
                          "host_shape_s": round(t_host_shape, 4), "device_bank_s": round(t_dev, 5),
                          "bank_MB": round(far.numel() * 16 / 1e6, 1), "rel_err_vs_host": err,
                          "host_threads": os.cpu_count()}))


if __name__ == "__main__":
    main()
