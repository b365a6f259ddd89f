"""ctypes bindings of the native libraries.

libfpbem_cuda.so carries the sm_100a kernels behind the C-ABI of
include/fpbem_cuda.h; libfpbem_host.so the host operator producer. There is
no fallback: if a library is missing or fails to load, this raises.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_DIR = Path(__file__).resolve().parent / "lib"

c_int_p = C.POINTER(C.c_int)
c_double_p = C.POINTER(C.c_double)


class NativeLibraryMissing(RuntimeError):
    pass


def _load(name: str) -> C.CDLL:
    path = LIB_DIR / name
    if not path.exists():
        raise NativeLibraryMissing(
            f"{path} is not built; run `python -m paper_2201_12050_b200.build` (or __graft_entry__.build())")
    return C.CDLL(str(path), mode=C.RTLD_GLOBAL)


class FmmDesc(C.Structure):
    """fpbem_cu_fmm_desc (include/fpbem_cuda.h)."""

    _fields_ = [
        ("counts", C.c_int * 3),
        ("n_dof", C.c_int),
        ("n_coef", C.c_int),
        ("n_near", C.c_int),
        ("near_offsets", C.c_void_p),
        ("near_blocks", C.c_void_p),
        ("u0", C.c_void_p),
        ("v0", C.c_void_p),
        ("fft_sizes", C.c_int * 3),
        ("lambda_", C.c_void_p),
        ("n_far", C.c_int),
        ("far_offsets", C.c_void_p),
        ("far_blocks", C.c_void_p),
        ("mirrored_level", C.c_int),
        ("max_rhs", C.c_int),
        ("n_hat", C.c_int),
        ("hat_indices", C.c_void_p),
        ("hat_blocks", C.c_void_p),
        ("n_far_hat", C.c_int),
        ("far_hat_indices", C.c_void_p),
        ("far_hat_blocks", C.c_void_p),
        ("lambda_hat", C.c_void_p),
        ("blocks_on_device", C.c_int),
        ("far_on_device", C.c_int),
        ("near_path", C.c_int),
        ("n_sym", C.c_int),
        ("sym_axes", C.c_void_p),
        ("sym_perms", C.c_void_p),
    ]


class Cell(C.Structure):
    """fpbem_cu_cell (include/fpbem_cuda.h)."""

    _fields_ = [
        ("n", C.c_int),
        ("corners", C.c_void_p),
        ("nv", C.c_void_p),
        ("centroid", C.c_void_p),
        ("normal", C.c_void_p),
        ("diameter", C.c_void_p),
        ("beta", C.c_void_p),
    ]


class C64(C.Structure):
    _fields_ = [("re", C.c_double), ("im", C.c_double)]


APPLY_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_size_t)

# every symbol include/fpbem_cuda.h declares (checked by tests/test_boundary.py)
CUDA_SYMBOLS = (
    "fpbem_cu_fmm_create", "fpbem_cu_fmm_destroy", "fpbem_cu_fmm_apply", "fpbem_cu_gmres",
    "fpbem_cu_gmres_fn", "fpbem_cu_fmm_bytes", "fpbem_cu_fmm_near_path", "fpbem_cu_spectrum", "fpbem_cu_set_stream",
    "fpbem_cu_get_stream", "fpbem_cu_far_info", "fpbem_cu_fmm_set_slabs", "fpbem_cu_fmm_slab_rows",
    "fpbem_cu_fmm_apply_slab", "fpbem_cu_fmm_slab_info",    "fpbem_cu_enable_stage_timing", "fpbem_cu_stage_times", "fpbem_cu_kernel_launches",
    "fpbem_cu_comm_unique_id", "fpbem_cu_comm_init", "fpbem_cu_comm_destroy", "fpbem_cu_fmm_set_comm",
    "fpbem_cu_comm_from_callback", "fpbem_cu_comm_simulated", "fpbem_cu_comm_traffic", "fpbem_cu_gmres_dist", "fpbem_cu_gmres_dist_rows",
    "fpbem_cu_fmm_set_partition", "fpbem_cu_fmm_partition", "fpbem_cu_fmm_far_pairs", "fpbem_cu_partition_pairs", "fpbem_cu_assemble_near", "fpbem_cu_assemble_hat",
    "fpbem_cu_m2l_bank", "fpbem_cu_evaluate_field", "fpbem_cu_last_error", "fpbem_cu_version",
)

_cuda = None
_host = None


def cuda() -> C.CDLL:
    global _cuda
    if _cuda is None:
        lib = _load("libfpbem_cuda.so")
        vp = C.c_void_p
        sig = {
            "fpbem_cu_fmm_create": (C.c_int, [C.POINTER(FmmDesc), C.c_int, C.POINTER(vp)]),
            "fpbem_cu_fmm_destroy": (None, [vp]),
            "fpbem_cu_fmm_apply": (C.c_int, [vp, vp, vp, C.c_int, C.c_int]),
            "fpbem_cu_gmres": (C.c_int, [vp, vp, vp, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, c_int_p,
                                         c_int_p, c_double_p, C.c_int, c_int_p]),
            "fpbem_cu_gmres_fn": (C.c_int, [C.c_int, C.c_longlong, APPLY_FN, vp, APPLY_FN, vp, vp, vp, C.c_double,
                                            C.c_int, C.c_int, C.c_int, c_int_p, c_int_p, c_double_p, C.c_int,
                                            c_int_p]),
            "fpbem_cu_fmm_bytes": (C.c_int, [vp, C.POINTER(C.c_size_t)]),
            "fpbem_cu_fmm_near_path": (C.c_int, [vp, c_int_p, c_int_p, C.POINTER(C.c_size_t), c_int_p, c_int_p,
                                                 c_double_p]),
            "fpbem_cu_spectrum": (C.c_int, [vp, c_int_p, vp]),
            "fpbem_cu_set_stream": (C.c_int, [vp, vp]),
            "fpbem_cu_get_stream": (C.c_int, [vp, C.POINTER(vp)]),
            "fpbem_cu_far_info": (C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
            "fpbem_cu_fmm_set_slabs": (C.c_int, [vp, vp]),
            "fpbem_cu_fmm_slab_rows": (C.c_int, [vp, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)]),
            "fpbem_cu_fmm_apply_slab": (C.c_int, [vp, vp, vp, C.c_int]),
            "fpbem_cu_fmm_slab_info": (C.c_int, [vp, C.POINTER(C.c_longlong)]),
            "fpbem_cu_enable_stage_timing": (C.c_int, [vp, C.c_int]),
            "fpbem_cu_stage_times": (C.c_int, [vp, c_double_p]),
            "fpbem_cu_kernel_launches": (C.c_longlong, [vp]),
            "fpbem_cu_comm_unique_id": (C.c_int, [C.c_char_p]),
            "fpbem_cu_comm_init": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(vp)]),
            "fpbem_cu_comm_destroy": (None, [vp]),
            "fpbem_cu_fmm_set_comm": (C.c_int, [vp, vp]),
            "fpbem_cu_comm_from_callback": (C.c_int, [ALLREDUCE_FN, vp, C.c_int, C.c_int, C.c_int, C.POINTER(vp)]),
            "fpbem_cu_comm_simulated": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(vp)]),
            "fpbem_cu_comm_traffic": (C.c_int, [vp, C.POINTER(C.c_ulonglong), C.POINTER(C.c_longlong), C.c_int]),
            "fpbem_cu_gmres_dist": (C.c_int, [vp, vp, vp, C.c_double, C.c_int, C.c_int, C.c_int, c_int_p, c_int_p,
                                              c_double_p, C.c_int, c_int_p]),
            "fpbem_cu_gmres_dist_rows": (C.c_int, [vp, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)]),
            "fpbem_cu_fmm_set_partition": (C.c_int, [vp, C.c_int, C.c_int, C.c_double]),
            "fpbem_cu_fmm_partition": (C.c_int, [vp, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong),
                                                 C.POINTER(C.c_double)]),
            "fpbem_cu_fmm_far_pairs": (C.c_int, [vp, C.POINTER(C.c_double)]),
            "fpbem_cu_partition_pairs": (C.c_int, [C.c_longlong, C.c_int, C.c_int, C.c_double, C.POINTER(C.c_longlong),
                                                   C.POINTER(C.c_longlong)]),
            "fpbem_cu_last_error": (C.c_char_p, []),
            "fpbem_cu_version": (C.c_char_p, []),
            "fpbem_cu_assemble_near": (C.c_int, [C.POINTER(Cell), C.c_double, C64, c_double_p, C.c_int, c_int_p,
                                                 C.c_int, C.c_int, C.c_double, C64, C.c_int, vp, C.c_int]),
            "fpbem_cu_assemble_hat": (C.c_int, [C.POINTER(Cell), C.c_double, C64, c_double_p, c_int_p, C.c_int,
                                                c_int_p, C.c_int, C.c_double, C64, C.c_int, vp, C.c_int]),
            "fpbem_cu_evaluate_field": (C.c_int, [C.POINTER(Cell), C.c_double, c_double_p, c_int_p, vp, C.c_int,
                                                  c_double_p, vp, C.c_int, C.c_double, C64, C.c_int, vp, C.c_int]),
            "fpbem_cu_m2l_bank": (C.c_int, [C.c_int, C.c_double, C.c_int, c_double_p, c_double_p, C.c_int, C64,
                                            C.c_int, vp, C.c_int]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _cuda = lib
    return _cuda


def host() -> C.CDLL:
    global _host
    if _host is None:
        lib = _load("libfpbem_host.so")
        vp = C.c_void_p
        sig = {
            "fh_last_error": (C.c_char_p, []),
            "fh_scene_create": (vp, [C.c_int, C.c_int]),
            "fh_scene_custom": (vp, [C.c_int, c_double_p, c_int_p, c_double_p, C.c_double]),
            "fh_scene_destroy": (None, [vp]),
            "fh_scene_info": (None, [vp, c_int_p, c_double_p]),
            "fh_scene_set_k": (None, [vp, C.c_double]),
            "fh_scene_set_halfspace": (None, [vp, C.c_int, C.c_double, C.c_double, C.c_double]),
            "fh_scene_shift_cell": (None, [vp, c_double_p]),
            "fh_fmm_image_arrays": (None, [vp] + [C.POINTER(vp)] * 4),
            "fh_scene_sweep": (None, [vp, c_double_p]),
            "fh_scene_set_sources": (None, [vp, C.c_int, c_int_p, c_double_p]),
            "fh_scene_rhs": (C.c_int, [vp, C.c_int, vp]),
            "fh_scene_incident": (C.c_int, [vp, C.c_int, C.c_int, c_double_p, vp]),
            "fh_scene_field": (C.c_int, [vp, C.c_int, vp, C.c_int, c_double_p, vp]),
            "fh_insertion_loss": (C.c_int, [C.c_int, vp, vp, vp]),
            "fh_scene_dense": (C.c_int, [vp, vp]),
            "fh_scene_cell": (C.c_int, [vp, c_double_p, c_double_p, c_double_p, c_double_p, c_double_p, c_int_p]),
            "fh_cell_symmetries": (C.c_int, [vp, c_int_p]),
            "fh_interaction_block": (C.c_int, [vp, c_double_p, C.c_int, vp]),
            "fh_classify": (C.c_int, [vp, c_int_p, c_int_p, c_int_p, c_int_p, C.c_int, c_double_p]),
            "fh_fmm_assemble": (vp, [vp, C.c_int, C.c_int]),
            "fh_fmm_destroy": (None, [vp]),
            "fh_fmm_info": (None, [vp, c_int_p]),
            "fh_fmm_arrays": (None, [vp] + [C.POINTER(vp)] * 6),
            "fh_sph_bessel": (None, [C.c_int, C.c_double, c_double_p, c_double_p]),
            "fh_wigner3j": (C.c_double, [C.c_int] * 6),
            "fh_solid_gradients": (C.c_int, [C.c_int, c_double_p, C.c_double, vp, vp, vp, vp]),
            "fh_solid_singular": (C.c_int, [C.c_int, c_double_p, C.c_double, vp]),
            "fh_m2l_block": (C.c_int, [C.c_int, c_double_p, C.c_double, vp]),
            "fh_expansions": (C.c_int, [vp, C.c_int, c_double_p, vp, vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _host = lib
    return _host
