"""First and repeated GMRES solve times of one configuration (restart 50, tol 1e-6)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    from paper_2201_12050_b200 import FmmOperators, Scene, gmres

    cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    sc = Scene(cid, 0)
    data = sc.assemble_fmm(4)
    op = FmmOperators(data)
    b = torch.from_numpy(sc.rhs(0)).cuda()
    for k in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        rep = gmres(op, b, tol=1e-6, restart=50, max_iter=1000)
        torch.cuda.synchronize()
        print(f"cfg{cid} solve {k}: {time.perf_counter() - t:.3f} s, {rep.iterations} iterations", flush=True)


if __name__ == "__main__":
    main()
