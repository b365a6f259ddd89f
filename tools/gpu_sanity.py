"""Quick GPU sanity run: GPU matvec / spectrum / GMRES vs the CPU oracle."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle as O  # noqa: E402
from paper_2201_12050_b200 import FmmOperators, Scene, gmres  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def main():
    rng = np.random.default_rng(0)
    for cid, var in [(1, 0), (2, 2), (3, 2), (4, 2), (5, 2), (6, 8)]:
        sc = Scene(cid, var)
        t = time.time()
        d = sc.assemble_fmm(4)
        ta = time.time() - t
        ora = O.OracleFmm(d)
        op = FmmOperators(d)
        sizes, lam = op.spectrum()
        p = rng.uniform(-1, 1, sc.N) + 1j * rng.uniform(-1, 1, sc.N)
        y = op.matvec(p)
        yo = ora.matvec(p)
        print(f"cfg{cid}/{var} counts={sc.counts} n={sc.n_dof} near={d.n_near} far={d.n_far} asm={ta:.2f}s "
              f"sizes={sizes}/{ora.sizes} lam_err={rel(lam, ora.lambda_):.2e} matvec_err={rel(y, yo):.2e} "
              f"bytes={op.stored_bytes()}", flush=True)
        b = sc.rhs(0)
        t = time.time()
        rep = gmres(op, b, tol=1e-6, restart=50, max_iter=300)
        tg = time.time() - t
        t = time.time()
        xo, its, conv, hist = ora.gmres(b, tol=1e-6, restart=50, max_iter=300)
        to = time.time() - t
        print(f"   gmres gpu its={rep.iterations} conv={rep.converged} t={tg:.2f}s | oracle its={its} conv={conv} "
              f"t={to:.2f}s | sol_err={rel(rep.solution, xo):.2e}", flush=True)


if __name__ == "__main__":
    main()
