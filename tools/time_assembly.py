"""Host vs device near-field assembly time for the BASELINE configs."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    from paper_2201_12050_b200 import Scene
    from paper_2201_12050_b200.fmm import assemble_near_gpu

    cfgs = [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "1,2,3,4,5").split(",")]
    for cid in cfgs:
        sc = Scene(cid, 0)
        t = time.perf_counter()
        shape = sc.assemble_fmm(4, skip_near_values=True)
        t_far = time.perf_counter() - t
        assemble_near_gpu(sc, shape)  # warm-up (module load, rules)
        torch.cuda.synchronize()
        t = time.perf_counter()
        blocks = assemble_near_gpu(sc, shape)
        torch.cuda.synchronize()
        t_gpu = time.perf_counter() - t
        t = time.perf_counter()
        full = sc.assemble_fmm(4)
        t_host = time.perf_counter() - t
        err = float(np.linalg.norm(blocks.cpu().numpy() - np.asarray(full.near_blocks)) /
                    np.linalg.norm(np.asarray(full.near_blocks)))
        entries = shape.n_near * shape.n_dof ** 2
        print(f"cfg{cid}: {entries / 1e6:.1f}M entries  host (16 threads, incl. far bank) {t_host:.2f} s  "
              f"far bank + U0/V0 only {t_far:.2f} s  device near blocks {t_gpu * 1e3:.1f} ms  "
              f"({entries / t_gpu / 1e9:.2f} G entries/s)  rel diff {err:.1e}", flush=True)


if __name__ == "__main__":
    main()
