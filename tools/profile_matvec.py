"""Profiling driver: a few FMM applies of one configuration on cuda:0.

    python tools/profile_matvec.py --config 2 [--synthetic] [--applies 5] [--nrhs 1]

--synthetic fills the operator with seeded random blocks of the config's exact
shapes (same offsets, n_dof, lattice) instead of assembling it, so profiling
runs do not pay the host assembly; kernel timings do not depend on values.
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


class Synthetic:
    def __init__(self, sc, n_t=4, seed=0):
        rng = np.random.default_rng(seed)
        near, far, _, _ = sc.classify()
        self.counts = sc.counts
        self.n_dof = sc.n_dof
        self.n_coef = (n_t + 1) ** 2
        n, b = self.n_dof, self.n_coef
        self.near_offsets = near
        self.far_offsets = far
        self.n_near, self.n_far = len(near), len(far)
        self.near_blocks = (rng.uniform(-1, 1, (len(near), n, n)) + 1j * rng.uniform(-1, 1, (len(near), n, n))) / n
        self.far_blocks = (rng.uniform(-1, 1, (len(far), b, b)) + 1j * rng.uniform(-1, 1, (len(far), b, b))) * 1e-3
        self.u0 = rng.uniform(-1, 1, (b, n)) + 0j
        self.v0 = rng.uniform(-1, 1, (n, b)) + 0j
        self.N = int(np.prod(self.counts)) * n


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--synthetic", action="store_true")
    ap.add_argument("--applies", type=int, default=5)
    ap.add_argument("--nrhs", type=int, default=1)
    args = ap.parse_args()
    import torch

    from paper_2201_12050_b200 import FmmOperators, Scene

    sc = Scene(args.config, args.variant)
    t = time.perf_counter()
    data = Synthetic(sc) if args.synthetic else sc.assemble_fmm(4)
    print(f"operator ready in {time.perf_counter() - t:.1f} s", file=sys.stderr)
    op = FmmOperators(data, max_rhs=args.nrhs)
    x = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, data.N * args.nrhs) + 0j).cuda()
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    op.set_stream(s.cuda_stream)
    op.enable_stage_timing(True)
    for _ in range(args.applies):
        y = op.matvec(x)
    torch.cuda.synchronize()
    st = op.stage_times()
    print({k: (v / max(1, st["applies"]) if k != "applies" else v) for k, v in st.items()})
    print("launches", op.kernel_launches(), "y norm", float(torch.linalg.vector_norm(y)))


if __name__ == "__main__":
    main()
