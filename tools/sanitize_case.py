"""A small end-to-end case for compute-sanitizer (memcheck / racecheck /
synccheck): one lattice-path product (pruned DFT passes, the DMMA mode product
with its bulk-copy ring, the pipelined M2L z kernel with its mbarrier ring),
a GMRES solve (the cooperative fused MGS with grid-wide syncs), the slab
product (one rank) and a direct-path product, each checked against the oracle.

    compute-sanitizer --tool memcheck python tools/sanitize_case.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import oracle as O
    from paper_2201_12050_b200 import FmmOperators, Scene, gmres

    rng = np.random.default_rng(7)
    sc = Scene(3, 2)  # 4 x 4 x 4 spheres: lattice near field, fused z kernel
    d = sc.assemble_fmm(4)
    ref = O.OracleFmm(d)
    x = rng.uniform(-1, 1, d.N) + 1j * rng.uniform(-1, 1, d.N)
    yo = ref.matvec(x)
    for path in ("lattice", "direct"):
        op = FmmOperators(d, near_path=path)
        y = op.matvec(x)
        err = np.linalg.norm(y - yo) / np.linalg.norm(yo)
        print(f"{path} product rel err {err:.2e}", flush=True)
        assert err < 1e-10
        if path == "lattice":
            rep = gmres(op, sc.rhs(0), tol=1e-6, restart=20, max_iter=60)
            print(f"gmres its {rep.iterations}", flush=True)
            op.set_slabs(None)
            ys = op.matvec_slab(x)
            err = np.linalg.norm(ys - yo) / np.linalg.norm(yo)
            print(f"slab product rel err {err:.2e}", flush=True)
            assert err < 1e-10
        op.close()
    print("sanitize case ok", flush=True)


if __name__ == "__main__":
    main()
