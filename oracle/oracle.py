"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes veneer over oracle/_build/liboracle.so, the CPU restatement of the
reference's hot path (fpbem_oracle.cpp cites the reference file:line of every
function). Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline /
--impl reference legs may import this module.

Block arrays use the reference's storage: each b x b block column-major, so a
numpy array of shape (n_blocks, b, b) holds block s as blk[s].T.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

_LIB = Path(__file__).resolve().parent / "_build" / "liboracle.so"
_lib = None
_ip = C.POINTER(C.c_int)
_dp = C.POINTER(C.c_double)
APPLY_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_longlong)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not _LIB.exists():
            from paper_2201_12050_b200 import build

            build.build_oracle()
        L = C.CDLL(str(_LIB))
        vp = C.c_void_p
        sig = {
            "oracle_last_error": (C.c_char_p, []),
            "oracle_num_threads": (C.c_int, []),
            "oracle_set_num_threads": (None, [C.c_int]),
            "oracle_fft_friendly": (C.c_int, [C.c_int]),
            "oracle_toeplitz_matvec": (C.c_int, [_ip, C.c_int, C.c_int, _ip, vp, vp, vp]),
            "oracle_toeplitz_expand_dense": (C.c_int, [_ip, C.c_int, C.c_int, _ip, vp, vp]),
            "oracle_hankel_matvec": (C.c_int, [_ip, C.c_int, C.c_int, C.c_int, _ip, vp, vp, vp]),
            "oracle_spectrum_build": (C.c_int, [_ip, C.c_int, C.c_int, _ip, vp, _ip, _ip, vp]),
            "oracle_spectrum_matvec": (C.c_int, [_ip, _ip, C.c_int, vp, vp, vp]),
            "oracle_dft3": (C.c_int, [vp, _ip, C.c_int, C.c_int]),
            "oracle_mirror_permute": (C.c_int, [_ip, C.c_int, C.c_int, vp, vp]),
            "oracle_fmm_create": (vp, [_ip, C.c_int, C.c_int, C.c_int, _ip, vp, vp, vp, _ip, vp]),
            "oracle_fmm_set_image": (C.c_int, [vp, C.c_int, C.c_int, _ip, vp, _ip, vp]),
            "oracle_fmm_destroy": (None, [vp]),
            "oracle_fmm_matvec": (C.c_int, [vp, vp, vp, C.c_int]),
            "oracle_gmres_cb": (C.c_int, [APPLY_CB, vp, APPLY_CB, vp, vp, vp, C.c_longlong, C.c_double, C.c_int,
                                          C.c_int, _ip, _ip, _dp, C.c_int, _ip]),
            "oracle_fmm_gmres": (C.c_int, [vp, vp, vp, C.c_double, C.c_int, C.c_int, _ip, _ip, _dp, C.c_int, _ip]),
        }
        for k, (r, a) in sig.items():
            f = getattr(L, k)
            f.restype = r
            f.argtypes = a
        _lib = L
    return _lib


def _i(a):
    a = np.ascontiguousarray(a, np.int32)
    return a, a.ctypes.data_as(_ip)


def _c(a):
    a = np.ascontiguousarray(a, np.complex128)
    return a, a.ctypes.data


def _check(rc: int) -> None:
    if rc:
        raise RuntimeError(lib().oracle_last_error().decode())


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def set_num_threads(n: int) -> None:
    lib().oracle_set_num_threads(int(n))


def fft_friendly(n: int) -> int:
    return int(lib().oracle_fft_friendly(int(n)))


def toeplitz_matvec(counts, offsets, blocks, p) -> np.ndarray:
    """BlockToeplitzMatrix::matvec (src/assembly.cpp:62-84)."""
    c, cp = _i(counts)
    o, op = _i(np.asarray(offsets).reshape(-1, 3))
    bl, bp = _c(blocks)
    b = bl.shape[-1]
    pv, pp = _c(p)
    y = np.zeros_like(pv)
    _check(lib().oracle_toeplitz_matvec(cp, b, len(o), op, bp, pp, y.ctypes.data))
    return y


def toeplitz_expand_dense(counts, offsets, blocks) -> np.ndarray:
    c, cp = _i(counts)
    o, op = _i(np.asarray(offsets).reshape(-1, 3))
    bl, bp = _c(blocks)
    b = bl.shape[-1]
    n = int(np.prod(c)) * b
    a = np.zeros((n, n), np.complex128, order="F")
    _check(lib().oracle_toeplitz_expand_dense(cp, b, len(o), op, bp, a.ctypes.data))
    return a


def hankel_matvec(counts, level, indices, blocks, p) -> np.ndarray:
    """BlockHankelMatrix::matvec (src/assembly.cpp:152-178)."""
    c, cp = _i(counts)
    ix, ipp = _i(np.asarray(indices).reshape(-1, 3))
    bl, bp = _c(blocks)
    pv, pp = _c(p)
    y = np.zeros_like(pv)
    _check(lib().oracle_hankel_matvec(cp, bl.shape[-1], level, len(ix), ipp, bp, pp, y.ctypes.data))
    return y


def spectrum_build(counts, offsets, blocks, sizes=None):
    """CirculantSpectrum constructor (src/structured.cpp:63-108) -> (sizes, lambda[q*b*b])."""
    c, cp = _i(counts)
    o, op = _i(np.asarray(offsets).reshape(-1, 3))
    bl, bp = _c(blocks)
    b = bl.shape[-1]
    si = None
    if sizes is not None:
        si_arr, si = _i(sizes)
    so = np.zeros(3, np.int32)
    _check(lib().oracle_spectrum_build(cp, b, len(o), op, bp, si, so.ctypes.data_as(_ip), None))
    lam = np.zeros(int(np.prod(so)) * b * b, np.complex128)
    _check(lib().oracle_spectrum_build(cp, b, len(o), op, bp, si, so.ctypes.data_as(_ip), lam.ctypes.data))
    return tuple(int(v) for v in so), lam


def spectrum_matvec(counts, sizes, b, lam, p) -> np.ndarray:
    """CirculantSpectrum::matvec (src/structured.cpp:122-166)."""
    c, cp = _i(counts)
    s, sp = _i(sizes)
    lv, lp = _c(lam)
    pv, pp = _c(p)
    y = np.zeros_like(pv)
    _check(lib().oracle_spectrum_matvec(cp, sp, int(b), lp, pp, y.ctypes.data))
    return y


def dft3(data, sizes, howmany: int, sign: int) -> np.ndarray:
    d = np.array(data, np.complex128, copy=True)
    s, sp = _i(sizes)
    _check(lib().oracle_dft3(d.ctypes.data, sp, int(howmany), int(sign)))
    return d


def mirror_permute(counts, level, b, p) -> np.ndarray:
    c, cp = _i(counts)
    pv, pp = _c(p)
    out = np.zeros_like(pv)
    _check(lib().oracle_mirror_permute(cp, level, b, pp, out.ctypes.data))
    return out


class OracleFmm:
    """FmmOperators::matvec restated on the CPU (src/fmm.cpp:246-271).
    data: FmmData-like; spectrum from `lambda_`+`sizes`, else built from the
    far bank with the reference's 7-smooth padding."""

    def __init__(self, data, sizes=None, lambda_=None):
        self._keep = [data]
        c, cp = _i(data.counts)
        no, nop = _i(np.asarray(data.near_offsets).reshape(-1, 3))
        nb, nbp = _c(data.near_blocks)
        u0, u0p = _c(data.u0)
        v0, v0p = _c(data.v0)
        if lambda_ is None:
            sizes, lambda_ = spectrum_build(data.counts, data.far_offsets, data.far_blocks, sizes)
        self.sizes = tuple(int(s) for s in sizes)
        sz, szp = _i(self.sizes)
        lam, lamp = _c(lambda_)
        self.lambda_ = lam
        self._keep += [c, no, nb, u0, v0, sz, lam]
        self.N = int(np.prod(data.counts)) * int(data.n_dof)
        self._h = C.c_void_p(lib().oracle_fmm_create(cp, int(data.n_dof), int(data.n_coef), len(no), nop, nbp, u0p,
                                                      v0p, szp, lamp))
        level = int(getattr(data, "mirrored_level", -1))
        if level >= 0:
            # S_hat (block Hankel) and the spectrum of K_hat P (src/structured.cpp:185-198):
            # offsets o = idx with o[level] = idx[level] - (M - 1)
            counts = tuple(int(c) for c in data.counts)
            hi, hip = _i(np.asarray(data.hat_indices).reshape(-1, 3))
            hb, hbp = _c(data.hat_blocks)
            offs = np.asarray(data.far_hat_indices, np.int32).reshape(-1, 3).copy()
            offs[:, level] -= counts[level] - 1
            isz, ilam = spectrum_build(counts, offs, data.far_hat_blocks)
            iszv, iszp = _i(isz)
            il, ilp = _c(ilam)
            self.image_sizes, self.image_lambda = isz, il
            self._keep += [hi, hb, iszv, il]
            _check(lib().oracle_fmm_set_image(self._h, level, len(hi), hip, hbp, iszp, ilp))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().oracle_fmm_destroy(self._h)
            self._h = None

    def matvec(self, p) -> np.ndarray:
        pv, pp = _c(p)
        nrhs = pv.size // self.N
        y = np.zeros_like(pv)
        _check(lib().oracle_fmm_matvec(self._h, pp, y.ctypes.data, nrhs))
        return y

    def gmres(self, b, tol=1e-4, restart=100, max_iter=1000):
        bv, bp = _c(b)
        x = np.zeros_like(bv)
        its, conv, hl = C.c_int(), C.c_int(), C.c_int()
        hist = np.zeros(max(1, max_iter))
        rc = lib().oracle_fmm_gmres(self._h, bp, x.ctypes.data, tol, restart, max_iter, C.byref(its), C.byref(conv),
                                    hist.ctypes.data_as(_dp), len(hist), C.byref(hl))
        _check(rc)
        return x, its.value, bool(conv.value), list(hist[: hl.value])


def gmres(apply, b, tol=1e-4, restart=100, max_iter=1000, preconditioner=None):
    """solver::gmres over a numpy callable (src/solver.cpp:21-123).
    Returns (x, iterations, converged, history); raises RuntimeError on a
    non-finite operator output, like checked_apply (src/solver.cpp:13-17)."""
    bv, bp = _c(b)
    n = bv.size
    errs = []

    def wrap(fn):
        def cb(_ctx, vp, wp, nn):
            try:
                v = np.ctypeslib.as_array(C.cast(vp, _dp), shape=(2 * nn,)).view(np.complex128)
                w = np.ctypeslib.as_array(C.cast(wp, _dp), shape=(2 * nn,)).view(np.complex128)
                w[:] = fn(v.copy())
                return 0
            except BaseException as e:
                errs.append(e)
                return 1

        return APPLY_CB(cb)

    a = wrap(apply)
    p = wrap(preconditioner) if preconditioner is not None else APPLY_CB()
    x = np.zeros_like(bv)
    its, conv, hl = C.c_int(), C.c_int(), C.c_int()
    hist = np.zeros(max(1, max_iter))
    rc = lib().oracle_gmres_cb(a, None, p, None, bp, x.ctypes.data, n, tol, restart, max_iter, C.byref(its),
                               C.byref(conv), hist.ctypes.data_as(_dp), len(hist), C.byref(hl))
    if errs:
        raise errs[0]
    _check(rc)
    return x, its.value, bool(conv.value), list(hist[: hl.value])
