import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle as O
from paper_2201_12050_b200 import FmmOperators, Scene
cid, var = int(sys.argv[1]), int(sys.argv[2])
sc = Scene(cid, var)
d = sc.assemble_fmm(4)
print("n", d.n_dof, "counts", d.counts, "near", d.n_near, "far", d.n_far, flush=True)
op = FmmOperators(d)
print("created", flush=True)
p = np.ones(sc.N, complex)
y = op.matvec(p)
print("matvec ok", np.linalg.norm(y - O.OracleFmm(d).matvec(p)) / np.linalg.norm(y), flush=True)
