"""In-tree build of the native libraries (no JIT cache: the .so files travel
with the repo snapshot to the GPU box).

    libfpbem_cuda.so  sm_100a kernels + the C-ABI of include/fpbem_cuda.h
    libfpbem_host.so  host C++ operator producer (mesh, quadrature, assembly)
    oracle/_build/liboracle.so  CPU restatement (test infrastructure only)
"""
from __future__ import annotations

import hashlib
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor
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
                "device_assembly.cu", "comm.cu", "gmres_dist.cu", "cellwise.cu", "slab.cu"]
HOST_SOURCES = ["geometry.cpp", "kernels.cpp", "specfun.cpp", "assembly.cpp", "postproc.cpp", "capi.cpp"]
# portable x86-64 ISA level: the GPU box CPU may differ from the build container's
CPU_FLAGS = ["-O3", "-march=x86-64-v3", "-fPIC", "-fopenmp", "-std=c++17"]
# the oracle's complex products without the C99 Annex G inf/NaN recovery call
# (__muldc3): identical results for finite operands, and vectorisable like
# Eigen's complex kernels in the reference
ORACLE_FLAGS = CPU_FLAGS + ["-fcx-limited-range"]


def _run(cmd: list[str]) -> None:
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("build failed: " + " ".join(cmd[:4]) + " ...")


def _digest(sources: list[Path], flags: list[str]) -> str:
    h = hashlib.sha256()
    for f in flags:
        h.update(f.encode() + b"\0")
    for s in sorted(sources):
        h.update(s.name.encode() + b"\0" + s.read_bytes())
    return h.hexdigest()


def _stale(target: Path, sources: list[Path], flags: list[str] = ()) -> bool:
    """Rebuild unless the target exists and its stamp holds the hash of the
    current sources and flags (content, not mtimes: a repo snapshot or a fresh
    checkout may carry an old binary with newer-looking timestamps, or the reverse)."""
    stamp = target.with_name(target.name + ".stamp")
    if not target.exists() or not stamp.exists():
        return True
    return stamp.read_text().strip() != _digest(sources, list(flags))


def _stamp(target: Path, sources: list[Path], flags: list[str] = ()) -> None:
    target.with_name(target.name + ".stamp").write_text(_digest(sources, list(flags)) + "\n")


def build_cuda(force: bool = False) -> Path:
    LIB.mkdir(exist_ok=True)
    out = LIB / "libfpbem_cuda.so"
    deps = [CSRC / s for s in CUDA_SOURCES] + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.hpp")) + [
        ROOT / "include" / "fpbem_cuda.h"]
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]
    if force or _stale(out, deps, flags):
        objs = [str(LIB / (Path(s).stem + ".o")) for s in CUDA_SOURCES]
        jobs = max(1, min(len(CUDA_SOURCES), os.cpu_count() or 1))
        with ThreadPoolExecutor(jobs) as ex:  # one nvcc per translation unit, in parallel
            list(ex.map(lambda so: _run([NVCC, *flags, "-c", str(CSRC / so[0]), "-o", so[1]]),
                        zip(CUDA_SOURCES, objs)))
        _run([NVCC, *ARCH, "-shared", "-o", str(out), *objs, "-ldl"])
        for o in objs:
            Path(o).unlink(missing_ok=True)
        _stamp(out, deps, flags)
    return out


def build_host(force: bool = False) -> Path:
    LIB.mkdir(exist_ok=True)
    out = LIB / "libfpbem_host.so"
    deps = [HOST / s for s in HOST_SOURCES] + list(HOST.glob("*.hpp")) + [CSRC / "gaunt.hpp"]
    if force or _stale(out, deps, CPU_FLAGS):
        _run(["g++", *CPU_FLAGS, "-shared", "-o", str(out), *[str(HOST / s) for s in HOST_SOURCES]])
        _stamp(out, deps, CPU_FLAGS)
    return out


def build_oracle(force: bool = False) -> Path:
    out_dir = ORACLE / "_build"
    out_dir.mkdir(exist_ok=True)
    out = out_dir / "liboracle.so"
    src = ORACLE / "fpbem_oracle.cpp"
    if force or _stale(out, [src], ORACLE_FLAGS):
        _run(["g++", *ORACLE_FLAGS, "-shared", "-o", str(out), str(src)])
        _stamp(out, [src], ORACLE_FLAGS)
    return out


def build_driver(force: bool = False) -> Path:
    """tools/cpp_scene_solve: the C++-only host -> C-ABI path (host assembly, shim, device solve)."""
    out = LIB / "cpp_scene_solve"
    src = ROOT / "tools" / "cpp_scene_solve.cpp"
    deps = [src, LIB / "libfpbem_host.so", LIB / "libfpbem_cuda.so", ROOT / "include" / "fpbem_cuda.hpp",
            ROOT / "include" / "fpbem_cuda.h"] + list(HOST.glob("*.hpp"))
    if force or _stale(out, deps, ["driver"]):
        _run(["g++", "-O2", "-std=c++17", "-I", str(ROOT / "include"), "-I", str(HOST), str(src), "-L", str(LIB),
              "-lfpbem_host", "-lfpbem_cuda", f"-Wl,-rpath,{LIB}", "-fopenmp", "-o", str(out)])
        _stamp(out, deps, ["driver"])
    return out


def build_all(force: bool = False) -> None:
    build_host(force)
    build_oracle(force)
    build_cuda(force)
    build_driver(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
    print("built:", *(str(p) for p in sorted(LIB.glob("*.so"))), ORACLE / "_build" / "liboracle.so")
