"""B200-native periodic fast-multipole BEM hot path (arXiv 2201.12050).

The GMRES matrix-vector product of the single-level periodic FMBEM — Toeplitz
near field, P2M/L2P expansions, far-field M2L as a lattice circulant
convolution — and the GMRES vector operations, as sm_100a CUDA kernels behind
the C-ABI of include/fpbem_cuda.h. Python here is a thin veneer for tests and
benchmarks; the host operator producer is C++ (host/), the product path is
CUDA (csrc/).
"""
from .fmm import FmmOperators, SolveReport, gmres  # noqa: F401
from .host import FmmData, Scene  # noqa: F401

__all__ = ["FmmOperators", "SolveReport", "gmres", "FmmData", "Scene"]
