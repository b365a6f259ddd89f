"""The drop-in boundary: libfpbem_cuda.so loads on a CPU-only box and exports
every symbol include/fpbem_cuda.h declares; the host and oracle libraries
load; the product path refuses to run without a GPU instead of falling back."""
import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "fpbem_cuda.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fpbem_cu_\w+)\s*\(", text)) - {"fpbem_cu_apply_fn"})


def test_header_declares_the_reference_entry_points():
    syms = declared_symbols()
    for s in ("fpbem_cu_fmm_create", "fpbem_cu_fmm_apply", "fpbem_cu_gmres", "fpbem_cu_fmm_bytes",
              "fpbem_cu_fmm_destroy", "fpbem_cu_last_error"):
        assert s in syms


def test_cuda_library_exports_every_declared_symbol():
    from paper_2201_12050_b200 import _native

    lib = _native.cuda()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_native.CUDA_SYMBOLS) | {"fpbem_cu_gmres_fn"} >= set(declared_symbols())


def test_cuda_library_is_sm100a():
    import subprocess

    so = ROOT / "paper_2201_12050_b200" / "lib" / "libfpbem_cuda.so"
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(so)], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", str(so)], capture_output=True, text=True).stdout
    assert "DMMA" in sass  # the near-field GEMM runs on the FP64 tensor cores


def test_version_and_error_calls_need_no_gpu():
    from paper_2201_12050_b200 import _native

    lib = _native.cuda()
    assert b"sm_100a" in lib.fpbem_cu_version()
    h = C.c_void_p()
    assert lib.fpbem_cu_fmm_create(None, 0, C.byref(h)) == 6  # FPBEM_CU_EINVAL
    assert b"null" in lib.fpbem_cu_last_error()


def test_m2l_bank_validates_before_touching_the_device():
    """fpbem_cu_m2l_bank rejects what TranslationTable::m2l rejects (evaluation
    at the singularity, src/specfun.cpp) with EINVAL, GPU or not."""
    import numpy as np

    from paper_2201_12050_b200 import _native

    lib = _native.cuda()
    out = np.zeros(25 * 25 * 2, np.complex128)
    zero = np.zeros(3)
    one = np.array([0.0, 0.0, 1.0])
    call = lambda n_t, k, d, im: lib.fpbem_cu_m2l_bank(  # noqa: E731
        n_t, k, 1, d.ctypes.data_as(_native.c_double_p) if d is not None else None,
        im.ctypes.data_as(_native.c_double_p) if im is not None else None, 2, _native.C64(1.0, 0.0), 0,
        out.ctypes.data, 0)
    assert call(4, 2.0, zero, None) == 6 and b"translation vector" in lib.fpbem_cu_last_error()
    assert call(4, 2.0, one, zero) == 6
    assert call(4, 2.0, None, None) == 6
    assert call(16, 2.0, one, None) == 6 and b"n_t" in lib.fpbem_cu_last_error()
    assert call(4, 0.0, one, None) == 6


def test_evaluate_field_validates_before_touching_the_device():
    from paper_2201_12050_b200 import _native

    lib = _native.cuda()
    pitch = (C.c_double * 3)(1, 1, 1)
    bad = (C.c_int * 3)(0, 1, 1)
    assert lib.fpbem_cu_evaluate_field(None, 1.0, pitch, bad, None, 0, None, None, 2, 0.0,
                                       _native.C64(0, 0), 0, None, 0) == 6  # null cell
    cell = _native.Cell()
    assert lib.fpbem_cu_evaluate_field(C.byref(cell), 1.0, pitch, bad, None, 0, None, None, 2, 0.0,
                                       _native.C64(0, 0), 0, None, 0) == 1  # EDIM: counts < 1


def test_host_and_oracle_libraries_load():
    import oracle
    from paper_2201_12050_b200 import _native

    assert _native.host().fh_wigner3j(1, 1, 0, 0, 0, 0) != 0.0
    assert oracle.fft_friendly(31) == 32


def test_product_path_fails_loudly_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2201_12050_b200 import FmmOperators, Scene

    d = Scene(1, 2).assemble_fmm(2)
    with pytest.raises(RuntimeError):
        FmmOperators(d)


def test_cpp_shim_compiles_links_and_maps_errors(tmp_path):
    """include/fpbem_cuda.hpp (the reference-side binding) builds against the .so;
    a bad descriptor surfaces as the reference's exception type."""
    import subprocess

    src = tmp_path / "shim.cpp"
    src.write_text(r'''
#include <complex>
#include <cstdio>
#include <vector>
#include "fpbem_cuda.hpp"
int main() {
  fpbem_cu_fmm_desc d{};
  d.counts[0] = 0;  // invalid lattice -> FPBEM_CU_EDIM -> std::invalid_argument (src/fmm.cpp:250 style)
  try {
    fpbem_cuda::DeviceFmm op(d, 0);
  } catch (const std::invalid_argument& e) {
    std::printf("invalid_argument: %s\n", e.what());
    return 0;
  } catch (const std::exception& e) {
    std::printf("other: %s\n", e.what());
    return 2;
  }
  return 1;
}
''')
    lib = ROOT / "paper_2201_12050_b200" / "lib"
    exe = tmp_path / "shim"
    subprocess.run(["g++", "-std=c++17", "-I", str(ROOT / "include"), str(src), "-L", str(lib), "-lfpbem_cuda",
                    f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "invalid_argument" in out.stdout
