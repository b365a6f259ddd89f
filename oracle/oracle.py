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
            "oracle_set_level1_parallel": (C.c_int, [C.c_int]),
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


class _NoNear:
    """FmmData view with the near field removed (the far-field part of
    FmmOperators::matvec alone: P2M -> CirculantSpectrum::matvec -> L2P)."""

    def __init__(self, data):
        self._d = data
        self.near_offsets = np.zeros((0, 3), np.int32)
        self.near_blocks = np.zeros((0,), np.complex128)
        self.hat_indices = np.zeros((0, 3), np.int32)
        self.hat_blocks = np.zeros((0,), np.complex128)

    def __getattr__(self, k):
        return getattr(self._d, k)


def toeplitz_matvec_blocked(counts, offsets, blocks, p, n) -> np.ndarray:
    """BlockToeplitzMatrix::matvec (src/assembly.cpp:62-84) regrouped for the
    CHECKER: per stored offset, in the stored order, one dense product over all
    of its valid targets (numpy/BLAS zgemm), added to the targets' sums. Every
    target still sums its offsets in the stored order; only the order inside a
    block product differs from the reference's GEMV per (target, offset), at
    rounding level. Used where the GEMV-per-pair restatement is too slow for
    hundreds of products (stated-size GMRES parity); single matvecs are checked
    against the restatement itself."""
    m0, m1, m2 = (int(c) for c in counts)
    blk = np.asarray(blocks, np.complex128).reshape(-1, n, n)  # blk[s] = S_s^T (column-major storage)
    X = np.asarray(p, np.complex128).reshape(m2, m1, m0, n)
    Y = np.zeros_like(X)
    for s, (ox, oy, oz) in enumerate(np.asarray(offsets, np.int64).reshape(-1, 3)):
        rng = []
        for o, m in ((oz, m2), (oy, m1), (ox, m0)):
            lo, hi = max(0, o), min(m, m + o)  # targets t with 0 <= t - o < m
            rng.append((lo, hi, o))
        if any(hi <= lo for lo, hi, _ in rng):
            continue
        (z0, z1, oz_), (y0, y1, oy_), (x0, x1, ox_) = rng
        src = X[z0 - oz_:z1 - oz_, y0 - oy_:y1 - oy_, x0 - ox_:x1 - ox_].reshape(-1, n)
        Y[z0:z1, y0:y1, x0:x1] += (src @ blk[s]).reshape(z1 - z0, y1 - y0, x1 - x0, n)
    return Y.reshape(-1)


class OracleFmmChecker:
    """CHECKER-ONLY fast form of FmmOperators::matvec for stated-size GMRES
    parity: the near field through toeplitz_matvec_blocked (per-offset BLAS
    products, multi-threaded), the far field (P2M, CirculantSpectrum::matvec,
    L2P, src/fmm.cpp:256-267) through the restatement in fpbem_oracle.cpp, and
    GMRES through the restatement's solver::gmres (src/solver.cpp:21-123) with
    this product as its ApplyFn. Not for half-space operators (the restatement
    covers those)."""

    def __init__(self, data, near: str = "blas"):
        if int(getattr(data, "mirrored_level", -1)) >= 0:
            raise ValueError("OracleFmmChecker: no half-space image terms")
        if near not in ("blas", "fft"):
            raise ValueError("OracleFmmChecker: near must be 'blas' or 'fft'")
        self.counts = tuple(int(c) for c in data.counts)
        self.n = int(data.n_dof)
        self.N = int(np.prod(self.counts)) * self.n
        self.near_offsets = np.asarray(data.near_offsets, np.int32).reshape(-1, 3)
        self.near_blocks = np.asarray(data.near_blocks, np.complex128).reshape(-1, self.n, self.n)
        self.far = OracleFmm(_NoNear(data))  # builds the spectrum with the restatement (src/structured.cpp:63-108)
        self.b = int(data.n_coef)
        self.v0t = np.asarray(data.v0, np.complex128).reshape(self.n, self.b)  # [j][i] = V0[i][j]
        self.u0t = np.asarray(data.u0, np.complex128).reshape(self.b, self.n)  # [m][i] = U0[i][m]
        q = int(np.prod(self.far.sizes))
        self.lam_t = self.far.lambda_.reshape(q, self.b, self.b).transpose(0, 2, 1)  # [q] = Λ_q (row-major view)
        self.matvecs = 0
        self.near_mode = near
        if near == "fft":
            self._near_spectrum()

    def _near_spectrum(self) -> None:
        """Near field by the convolution theorem (CHECKER for many products over
        many offsets, e.g. cfg2's 125): the S_o embedded at slot o mod Ln with
        Ln_d = M_d + max|o_d| (no aliasing into the kept targets) and DFT'd once
        over the lattice axes (scipy.fft, multi-threaded); each product is then a
        pruned forward DFT, one n x n GEMV per mode and an inverse DFT."""
        import scipy.fft as sf

        R = np.abs(self.near_offsets).max(axis=0) if len(self.near_offsets) else np.zeros(3, int)
        self.nl = tuple(int(m + r) if m > 1 else 1 for m, r in zip(self.counts, R))  # (Lx, Ly, Lz)
        lx, ly, lz = self.nl
        n = self.n
        Sh = np.zeros((lz, ly, lx, n, n), np.complex128)
        for s, (ox, oy, oz) in enumerate(self.near_offsets):
            Sh[oz % lz, oy % ly, ox % lx] = self.near_blocks[s].T  # S_o (row = target)
        self.Sh = sf.fftn(Sh, axes=(0, 1, 2), workers=-1, overwrite_x=True).reshape(-1, n, n)

    def near_matvec(self, p) -> np.ndarray:
        if self.near_mode == "blas":
            return toeplitz_matvec_blocked(self.counts, self.near_offsets, self.near_blocks, p, self.n)
        import scipy.fft as sf

        m0, m1, m2 = self.counts
        lx, ly, lz = self.nl
        X = np.zeros((lz, ly, lx, self.n), np.complex128)
        X[:m2, :m1, :m0] = p.reshape(m2, m1, m0, self.n)
        Xh = sf.fftn(X, axes=(0, 1, 2), workers=-1).reshape(-1, self.n, 1)
        Yh = np.matmul(self.Sh, Xh).reshape(lz, ly, lx, self.n)
        Y = sf.ifftn(Yh, axes=(0, 1, 2), workers=-1)
        return np.ascontiguousarray(Y[:m2, :m1, :m0]).reshape(-1)

    def far_matvec(self, p) -> np.ndarray:
        """U0 IFFT(Λ FFT(pad(V0 p))) (src/fmm.cpp:256-267, src/structured.cpp:122-166)
        with multi-threaded transforms (scipy.fft workers) on the restatement's Λ."""
        import scipy.fft as sf

        m0, m1, m2 = self.counts
        lx, ly, lz = self.far.sizes
        P = p.reshape(-1, self.n)
        mom = P @ self.v0t  # (cells, b): M_c = V0 p_c
        field = np.zeros((lz, ly, lx, self.b), np.complex128)
        field[:m2, :m1, :m0] = mom.reshape(m2, m1, m0, self.b)
        F = sf.fftn(field, axes=(0, 1, 2), workers=-1).reshape(-1, self.b, 1)  # unnormalised, sign -1
        img = np.matmul(self.lam_t, F).reshape(lz, ly, lx, self.b)
        back = sf.ifftn(img, axes=(0, 1, 2), workers=-1)  # sign +1 and the 1/q of :156-164
        loc = np.ascontiguousarray(back[:m2, :m1, :m0]).reshape(-1, self.b)
        return (loc @ self.u0t).reshape(-1)

    def matvec(self, p) -> np.ndarray:
        p = np.ascontiguousarray(p, np.complex128)
        out = []
        for r in range(p.size // self.N):
            pr = p[r * self.N:(r + 1) * self.N]
            y = self.near_matvec(pr)
            y += self.far_matvec(pr)
            out.append(y)
            self.matvecs += 1
        return np.concatenate(out) if len(out) > 1 else out[0]

    def gmres(self, b, tol=1e-4, restart=100, max_iter=1000):
        prev = lib().oracle_set_level1_parallel(1)
        try:
            return gmres(self.matvec, b, tol=tol, restart=restart, max_iter=max_iter)
        finally:
            lib().oracle_set_level1_parallel(prev)
