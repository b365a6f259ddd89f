"""GMRES solution agreement with the oracle per near-field path (scene (2, 2),
restart 10): direct, lattice storing every mode, lattice with symmetry orbits."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle as O  # noqa: E402
from paper_2201_12050_b200 import FmmOperators, Scene, gmres  # noqa: E402

cid, var, restart = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (2, 2, 10)))
sc = Scene(cid, var)
d = sc.assemble_fmm(4)
b = sc.rhs(0)
x, its, conv, hist = O.OracleFmm(d).gmres(b, tol=1e-6, restart=restart, max_iter=2000)
print("oracle", its, conv)
for name, kw in (("direct", dict(near_path="direct")), ("lattice", dict(near_path="lattice", use_symmetries=False)),
                 ("lattice+sym", dict(near_path="lattice"))):
    op = FmmOperators(d, **kw)
    rep = gmres(op, b, tol=1e-6, restart=restart, max_iter=2000)
    p = np.random.default_rng(1).uniform(-1, 1, d.N) + 0j
    mv = np.linalg.norm(op.matvec(p) - O.OracleFmm(d).matvec(p)) / np.linalg.norm(O.OracleFmm(d).matvec(p))
    print(name, op.near_path()[:4], rep.iterations, rep.converged, "sol rel", np.linalg.norm(rep.solution - x) / np.linalg.norm(x),
          "matvec rel", mv)
