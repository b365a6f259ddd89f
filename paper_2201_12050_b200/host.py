"""Python veneer over the host operator producer (libfpbem_host.so).

Scene mirrors the reference's scene set-up (src/scene.cpp:258-289: cell mesh,
lattice, incident field, WaveContext); FmmData mirrors the data members of
FmmOperators (include/fpbem/fmm.hpp:54-71) as produced by
assemble_periodic_fmm (src/fmm.cpp:125-190), minus the spectrum, which the
device builds from the far M2L bank.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native

CONFIGS = {1: "cfg1", 2: "cfg2", 3: "cfg3", 4: "cfg4", 5: "cfg5"}


def _err() -> str:
    return _native.host().fh_last_error().decode()


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_native.c_double_p)


def _ip(a: np.ndarray):
    return a.ctypes.data_as(_native.c_int_p)


class Scene:
    """One BASELINE.json configuration (config_id 1..5; variant 0 as stated,
    1 reference-pinned quad variant, 2 shrunk lattice for fast checks), or a
    custom cell via Scene.custom."""

    def __init__(self, config_id: int = 1, variant: int = 0, _handle=None):
        lib = _native.host()
        h = _handle if _handle is not None else lib.fh_scene_create(config_id, variant)
        if not h:
            raise ValueError(_err())
        self._h = C.c_void_p(h)
        self.config_id = config_id
        self.variant = variant
        self.halfspace = None  # (axis, offset, reflection) once set_halfspace activates one

    @classmethod
    def custom(cls, kind: str, params, counts, pitch, k: float) -> "Scene":
        kinds = {"cube_sphere": 0, "icosphere": 1, "cylinder": 2, "box": 3, "wall": 4}
        p = np.asarray(params, dtype=np.float64)
        c = np.asarray(counts, dtype=np.int32)
        pt = np.asarray(pitch, dtype=np.float64)
        h = _native.host().fh_scene_custom(kinds[kind], _dp(p), _ip(c), _dp(pt), float(k))
        if not h:
            raise ValueError(_err())
        return cls(0, 0, _handle=h)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _native.host().fh_scene_destroy(h)
            self._h = None

    def _info(self):
        info = np.zeros(6, np.int32)
        dinfo = np.zeros(4, np.float64)
        _native.host().fh_scene_info(self._h, _ip(info), _dp(dinfo))
        return info, dinfo

    @property
    def counts(self) -> tuple[int, int, int]:
        return tuple(int(v) for v in self._info()[0][:3])

    @property
    def pitch(self) -> tuple[float, float, float]:
        return tuple(float(v) for v in self._info()[1][:3])

    @property
    def n_dof(self) -> int:
        return int(self._info()[0][3])

    @property
    def n_cells(self) -> int:
        c = self.counts
        return c[0] * c[1] * c[2]

    @property
    def N(self) -> int:
        return self.n_cells * self.n_dof

    @property
    def n_rhs(self) -> int:
        return int(self._info()[0][4])

    @property
    def wavenumber(self) -> float:
        return float(self._info()[1][3])

    @wavenumber.setter
    def wavenumber(self, k: float) -> None:
        _native.host().fh_scene_set_k(self._h, float(k))

    def set_halfspace(self, axis: int, offset: float, reflection: complex) -> None:
        """Mirror plane x_axis = offset with a complex reflection coefficient
        (geometry.hpp:66-78); reflection 0 switches it off."""
        r = complex(reflection)
        _native.host().fh_scene_set_halfspace(self._h, int(axis), float(offset), r.real, r.imag)
        self.halfspace = (int(axis), float(offset), r) if r != 0 else None

    def incident(self, points, field: int = 0) -> np.ndarray:
        """incident_values(field, x, .).first at each point, with the half-space
        image sources (src/kernels.cpp:305-325)."""
        pts = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
        out = np.zeros(len(pts), np.complex128)
        if _native.host().fh_scene_incident(self._h, field, len(pts), _dp(pts), out.ctypes.data):
            raise ValueError(_err())
        return out

    def field_host(self, solution, points, field: int = 0) -> np.ndarray:
        """postproc::evaluate_field on the host (src/postproc.cpp:39-62), all
        host threads: the checker for fmm.evaluate_field_gpu."""
        pts = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
        sol = np.ascontiguousarray(solution, np.complex128)
        if sol.size != self.N:
            raise ValueError("evaluate_field: solution length mismatch")
        out = np.zeros(len(pts), np.complex128)
        if _native.host().fh_scene_field(self._h, field, sol.ctypes.data, len(pts), _dp(pts), out.ctypes.data):
            raise ValueError(_err())
        return out

    def shift_cell(self, shift) -> None:
        s = np.asarray(shift, np.float64)
        _native.host().fh_scene_shift_cell(self._h, _dp(s))

    def sweep_hz(self) -> list[float]:
        n = int(self._info()[0][5])
        out = np.zeros(max(n, 1), np.float64)
        _native.host().fh_scene_sweep(self._h, _dp(out))
        return [float(v) for v in out[:n]]

    def set_sources(self, kinds, vecs) -> None:
        """kinds: 1 plane wave (direction), 0 monopole (position), one field each."""
        k = np.asarray(kinds, np.int32)
        v = np.ascontiguousarray(vecs, np.float64).reshape(-1, 3)
        _native.host().fh_scene_set_sources(self._h, len(k), _ip(k), _dp(v))

    def rhs(self, field: int = 0) -> np.ndarray:
        """assemble_rhs: p_inc + alpha dp_inc/dn at the collocation points (src/assembly.cpp:241-251)."""
        out = np.zeros(self.N, np.complex128)
        if _native.host().fh_scene_rhs(self._h, field, out.ctypes.data):
            raise ValueError(_err())
        return out

    def dense(self) -> np.ndarray:
        """Dense collocation matrix of the replicated mesh (src/assembly.cpp:253-276)."""
        n = self.N
        out = np.zeros((n, n), np.complex128, order="F")
        if _native.host().fh_scene_dense(self._h, out.ctypes.data):
            raise ValueError(_err())
        return out

    def cell(self) -> dict:
        n = self.n_dof
        d = dict(corners=np.zeros((n, 4, 3)), centroid=np.zeros((n, 3)), normal=np.zeros((n, 3)),
                 area=np.zeros(n), diameter=np.zeros(n), nv=np.zeros(n, np.int32))
        if _native.host().fh_scene_cell(self._h, _dp(d["corners"]), _dp(d["centroid"]), _dp(d["normal"]),
                                        _dp(d["area"]), _dp(d["diameter"]), _ip(d["nv"])):
            raise ValueError(_err())
        return d

    def cell_symmetries(self) -> list[tuple[int, np.ndarray]]:
        """Axis sign maps g of the unit cell (bit d of g flips axis d about the
        bounding-box centre: mirrors, half-turns, the inversion) that map the
        mesh onto itself, with the element permutation P_g of each (P_g[j] =
        the element whose corners are j's mapped corners); [] when the cell has
        none. Extension: the lattice near field stores one
        block per orbit of Fourier modes after checking
        S_{A_g o}[P_g i, P_g j] = S_o[i, j] on the device. Cached."""
        if not hasattr(self, "_symmetries"):
            n = self.n_dof
            perms = np.zeros((8, n), np.int32)
            mask = _native.host().fh_cell_symmetries(self._h, _ip(perms))
            if mask < 0:
                raise ValueError(_err())
            self._symmetries = [(g, perms[g].copy()) for g in range(1, 8) if mask >> g & 1]
        return self._symmetries

    def interaction_block(self, shift, self_terms: bool) -> np.ndarray:
        n = self.n_dof
        out = np.zeros((n, n), np.complex128, order="F")
        s = np.asarray(shift, np.float64)
        if _native.host().fh_interaction_block(self._h, _dp(s), int(self_terms), out.ctypes.data):
            raise ValueError(_err())
        return out

    def classify(self):
        """(near offsets, far offsets, base_center, radius) — make_box_grid/admissible
        over the offset loop (src/fmm.cpp:156-179, src/geometry.cpp:180-196)."""
        nn = C.c_int()
        nf = C.c_int()
        grid = np.zeros(4)
        lib = _native.host()
        lib.fh_classify(self._h, C.byref(nn), C.byref(nf), None, None, 0, _dp(grid))
        cap = max(nn.value, nf.value, 1)
        near = np.zeros((cap, 3), np.int32)
        far = np.zeros((cap, 3), np.int32)
        lib.fh_classify(self._h, C.byref(nn), C.byref(nf), _ip(near), _ip(far), cap, _dp(grid))
        return near[: nn.value].copy(), far[: nf.value].copy(), grid[:3].copy(), float(grid[3])

    def expansions(self, n_t: int, center) -> tuple[np.ndarray, np.ndarray]:
        n, b = self.n_dof, (n_t + 1) ** 2
        u0 = np.zeros((n, b), np.complex128, order="F")
        v0 = np.zeros((b, n), np.complex128, order="F")
        c = np.asarray(center, np.float64)
        if _native.host().fh_expansions(self._h, n_t, _dp(c), u0.ctypes.data, v0.ctypes.data):
            raise ValueError(_err())
        return u0, v0

    def assemble_fmm(self, n_t: int = 4, skip_near_values: bool = False, skip_far_values: bool = False) -> "FmmData":
        """assemble_periodic_fmm on the host. skip_near_values / skip_far_values
        leave the near (S, S_hat) / far (K bank, K_hat) values empty for
        device assembly (fmm.assemble_near_gpu / fmm.assemble_far_gpu)."""
        h = _native.host().fh_fmm_assemble(self._h, n_t, int(bool(skip_near_values)) | (int(bool(skip_far_values)) << 1))
        if not h:
            raise ValueError(_err())
        data = FmmData(h)
        data.cell_symmetries = self.cell_symmetries()
        return data


class FmmData:
    """Host-assembled operator data. Arrays are zero-copy views into the native
    handle (kept alive by this object)."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle)
        lib = _native.host()
        info = np.zeros(12, np.int32)
        lib.fh_fmm_info(self._h, _ip(info))
        self.counts = tuple(int(v) for v in info[:3])
        self.n_dof = int(info[3])
        self.n_coef = int(info[4])
        self.n_near = int(info[5])
        self.n_far = int(info[6])
        self.has_near_values = bool(info[7])
        ptrs = [C.c_void_p() for _ in range(6)]
        lib.fh_fmm_arrays(self._h, *[C.byref(p) for p in ptrs])
        n, b = self.n_dof, self.n_coef

        def view(p, count, dtype, shape):
            if count == 0 or not p.value:
                return np.zeros(shape, dtype)
            buf = (C.c_char * (count * np.dtype(dtype).itemsize)).from_address(p.value)
            buf._owner = self  # the views keep the native handle alive
            return np.frombuffer(buf, dtype=dtype).reshape(shape)

        self.near_offsets = view(ptrs[0], 3 * self.n_near, np.int32, (self.n_near, 3))
        # block s is column-major n x n: reshape (s, col, row)
        self.near_blocks = view(ptrs[1], self.n_near * n * n if self.has_near_values else 0, np.complex128,
                                (self.n_near, n, n) if self.has_near_values else (0, n, n))
        self.far_offsets = view(ptrs[2], 3 * self.n_far, np.int32, (self.n_far, 3))
        self.has_far_values = bool(info[11])
        nf = self.n_far if self.has_far_values else 0
        self.far_blocks = view(ptrs[3], nf * b * b, np.complex128, (nf, b, b))
        self.u0 = view(ptrs[4], n * b, np.complex128, (b, n))  # column-major n x b -> (col, row)
        self.v0 = view(ptrs[5], n * b, np.complex128, (n, b))  # column-major b x n -> (col, row)
        # half-space image pair (block Hankel along mirrored_level; -1 = none)
        self.mirrored_level = int(info[8])
        self.n_hat, self.n_far_hat = int(info[9]), int(info[10])
        iptrs = [C.c_void_p() for _ in range(4)]
        lib.fh_fmm_image_arrays(self._h, *[C.byref(p) for p in iptrs])
        nh = self.n_hat if self.has_near_values else 0
        self.hat_indices = view(iptrs[0], 3 * self.n_hat, np.int32, (self.n_hat, 3))
        self.hat_blocks = view(iptrs[1], nh * n * n, np.complex128, (nh, n, n))
        self.far_hat_indices = view(iptrs[2], 3 * self.n_far_hat, np.int32, (self.n_far_hat, 3))
        nfh = self.n_far_hat if self.has_far_values else 0
        self.far_hat_blocks = view(iptrs[3], nfh * b * b, np.complex128, (nfh, b, b))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _native.host().fh_fmm_destroy(h)
            self._h = None

    @property
    def n_cells(self) -> int:
        return self.counts[0] * self.counts[1] * self.counts[2]

    @property
    def N(self) -> int:
        return self.n_cells * self.n_dof


def insertion_loss(p_inc, p) -> float:
    """postproc::insertion_loss (src/postproc.cpp:64-72): 20 log10(sum|p_inc| / sum|p|)."""
    a = np.ascontiguousarray(p_inc, np.complex128)
    b = np.ascontiguousarray(p, np.complex128)
    il = C.c_double()
    if a.size != b.size or _native.host().fh_insertion_loss(a.size, a.ctypes.data, b.ctypes.data, C.byref(il)):
        raise ValueError(_err() if a.size == b.size else "insertion_loss: paired non-empty vectors required")
    return float(il.value)


def grid_points(lo, hi, counts) -> np.ndarray:
    """postproc::grid_points (src/postproc.cpp:118-133): z slowest, x fastest;
    a single-point axis sits at the midpoint."""
    lo = np.asarray(lo, np.float64)
    hi = np.asarray(hi, np.float64)
    if any(c < 1 for c in counts):
        raise ValueError("grid_points: counts must be >= 1")
    axes = [np.array([0.5 * (lo[d] + hi[d])]) if counts[d] == 1 else
            lo[d] + (hi[d] - lo[d]) * np.arange(counts[d]) / (counts[d] - 1.0) for d in range(3)]
    z, y, x = np.meshgrid(axes[2], axes[1], axes[0], indexing="ij")
    return np.stack([x.ravel(), y.ravel(), z.ravel()], axis=1)


def m2l_block(n_t: int, delta, k: float) -> np.ndarray:
    b = (n_t + 1) ** 2
    out = np.zeros((b, b), np.complex128, order="F")
    d = np.asarray(delta, np.float64)
    if _native.host().fh_m2l_block(n_t, _dp(d), float(k), out.ctypes.data):
        raise ValueError(_err())
    return out


def sph_bessel(n_max: int, x: float):
    j = np.zeros(n_max + 1)
    y = np.zeros(n_max + 1)
    _native.host().fh_sph_bessel(n_max, float(x), _dp(j), _dp(y) if x > 0 else None)
    return j, y


def wigner3j(j1, j2, j3, m1, m2, m3) -> float:
    return float(_native.host().fh_wigner3j(j1, j2, j3, m1, m2, m3))


def solid_regular_gradients(n_max: int, v, k: float):
    cnt = (n_max + 1) ** 2
    arrs = [np.zeros(cnt, np.complex128) for _ in range(4)]
    vv = np.asarray(v, np.float64)
    if _native.host().fh_solid_gradients(n_max, _dp(vv), float(k), *[a.ctypes.data for a in arrs]):
        raise ValueError(_err())
    return arrs


def solid_singular(n_max: int, v, k: float) -> np.ndarray:
    out = np.zeros((n_max + 1) ** 2, np.complex128)
    vv = np.asarray(v, np.float64)
    if _native.host().fh_solid_singular(n_max, _dp(vv), float(k), out.ctypes.data):
        raise ValueError(_err())
    return out
