"""In-tree build of the native libraries (no JIT cache: the .so files travel
with the repo snapshot to the GPU box).

    libfpbem_cuda.so  sm_100a kernels + the C-ABI of include/fpbem_cuda.h
    libfpbem_host.so  host C++ operator producer (mesh, quadrature, assembly)
    oracle/_build/liboracle.so  CPU restatement (test infrastructure only)
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
LIB = PKG / "lib"
CSRC = PKG / "csrc"
HOST = PKG / "host"
ORACLE = ROOT / "oracle"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUDA_SOURCES = ["near_field.cu", "m2l.cu", "krylov.cu", "assembly.cu", "far_bank.cu", "fpbem_cuda.cu", "gmres.cu",
                "device_assembly.cu", "comm.cu", "gmres_dist.cu"]
HOST_SOURCES = ["geometry.cpp", "kernels.cpp", "specfun.cpp", "assembly.cpp", "postproc.cpp", "capi.cpp"]
# portable x86-64 ISA level: the GPU box CPU may differ from the build container's
CPU_FLAGS = ["-O3", "-march=x86-64-v3", "-fPIC", "-fopenmp", "-std=c++17"]


def _run(cmd: list[str]) -> None:
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("build failed: " + " ".join(cmd[:4]) + " ...")


def _stale(target: Path, sources: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(s.stat().st_mtime > t for s in sources)


def build_cuda(force: bool = False) -> Path:
    LIB.mkdir(exist_ok=True)
    out = LIB / "libfpbem_cuda.so"
    deps = [CSRC / s for s in CUDA_SOURCES] + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.hpp")) + [
        ROOT / "include" / "fpbem_cuda.h"]
    if force or _stale(out, deps):
        objs = []
        for s in CUDA_SOURCES:
            obj = LIB / (Path(s).stem + ".o")
            _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                  "-c", str(CSRC / s), "-o", str(obj)])
            objs.append(str(obj))
        _run([NVCC, *ARCH, "-shared", "-o", str(out), *objs, "-ldl"])
        for o in objs:
            Path(o).unlink(missing_ok=True)
    return out


def build_host(force: bool = False) -> Path:
    LIB.mkdir(exist_ok=True)
    out = LIB / "libfpbem_host.so"
    deps = [HOST / s for s in HOST_SOURCES] + list(HOST.glob("*.hpp")) + [CSRC / "gaunt.hpp"]
    if force or _stale(out, deps):
        _run(["g++", *CPU_FLAGS, "-shared", "-o", str(out), *[str(HOST / s) for s in HOST_SOURCES]])
    return out


def build_oracle(force: bool = False) -> Path:
    out_dir = ORACLE / "_build"
    out_dir.mkdir(exist_ok=True)
    out = out_dir / "liboracle.so"
    src = ORACLE / "fpbem_oracle.cpp"
    if force or _stale(out, [src]):
        _run(["g++", *CPU_FLAGS, "-shared", "-o", str(out), str(src)])
    return out


def build_driver(force: bool = False) -> Path:
    """tools/cpp_scene_solve: the C++-only host -> C-ABI path (host assembly, shim, device solve)."""
    out = LIB / "cpp_scene_solve"
    src = ROOT / "tools" / "cpp_scene_solve.cpp"
    deps = [src, LIB / "libfpbem_host.so", LIB / "libfpbem_cuda.so", ROOT / "include" / "fpbem_cuda.hpp",
            ROOT / "include" / "fpbem_cuda.h"] + list(HOST.glob("*.hpp"))
    if force or _stale(out, deps):
        _run(["g++", "-O2", "-std=c++17", "-I", str(ROOT / "include"), "-I", str(HOST), str(src), "-L", str(LIB),
              "-lfpbem_host", "-lfpbem_cuda", f"-Wl,-rpath,{LIB}", "-fopenmp", "-o", str(out)])
    return out


def build_all(force: bool = False) -> None:
    build_host(force)
    build_oracle(force)
    build_cuda(force)
    build_driver(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
    print("built:", *(str(p) for p in sorted(LIB.glob("*.so"))), ORACLE / "_build" / "liboracle.so")
