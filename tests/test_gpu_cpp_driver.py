"""The C++-only drop-in path (tools/cpp_scene_solve.cpp): host C++ assembly ->
fpbem_cu_fmm_desc (with the cell's symmetries) -> the C-ABI shim -> device
product and device GMRES, compared with the oracle on the same scene and input
(matvec relative L2 <= 1e-10, iterations within +-1, solution <= 1e-8)."""
import subprocess

import numpy as np
import pytest

import oracle as O
from conftest import ROOT, rel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cid,var", [(1, 0), (3, 2), (5, 2)])
def test_cpp_host_to_device_solve_matches_oracle(tmp_path, cid, var):
    from paper_2201_12050_b200 import Scene
    from paper_2201_12050_b200.build import build_driver

    exe = build_driver()
    sc = Scene(cid, var)
    d = sc.assemble_fmm(4)
    rng = np.random.default_rng(cid)
    x = rng.uniform(-1, 1, d.N) + 1j * rng.uniform(-1, 1, d.N)
    xf, yf, sf = tmp_path / "x.bin", tmp_path / "y.bin", tmp_path / "s.bin"
    x.astype(np.complex128).tofile(xf)
    out = subprocess.run([str(exe), str(cid), str(var), str(xf), str(yf), str(sf)], capture_output=True, text=True,
                         cwd=ROOT, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    fields = out.stdout.split()
    info = dict(zip(fields[0::2], fields[1::2]))
    ora = O.OracleFmm(d)
    assert rel(np.fromfile(yf, np.complex128), ora.matvec(x)) <= 1e-10
    xo, its, conv, _ = ora.gmres(sc.rhs(0), tol=1e-6, restart=50, max_iter=1000)
    assert int(info["converged"]) == int(conv) and abs(int(info["iterations"]) - its) <= 1
    assert rel(np.fromfile(sf, np.complex128), xo) <= 1e-8
