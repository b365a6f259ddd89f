"""GPU-backed FmmOperators and GMRES — the reference-facing API of the hot path.

Mirrors fpbem::fmm::FmmOperators::matvec (include/fpbem/fmm.hpp:69,
src/fmm.cpp:246-271) and fpbem::solver::gmres / SolveReport / GmresOptions
(include/fpbem/solver.hpp:14-33, src/solver.cpp:21-123), with the same
argument meaning and error behaviour: a dimension mismatch raises ValueError
(std::invalid_argument), a non-finite operator output raises RuntimeError
("gmres: operator returned a non-finite value"), non-convergence is reported
in the SolveReport, not raised. All arithmetic runs in libfpbem_cuda.so on
the GPU; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native

OK, EDIM, ENONFINITE, ECUDA, ENOMEM, ENCCL, EINVAL = range(7)
PTR_HOST, PTR_DEVICE = 0, 1


def _raise(code: int) -> None:
    if code == OK:
        return
    msg = _native.cuda().fpbem_cu_last_error().decode()
    if code == EDIM:
        raise ValueError(msg)
    raise RuntimeError(msg)


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


class _TorchOrdered:
    """Orders a library stream against torch's current stream around a
    device-pointer call: the library waits for torch's producers of the inputs,
    and torch's stream waits for the library's work before anything enqueued
    after the call, so memory the caching allocator recycles (on this stream)
    is reused only after the library is done with it. (No record_stream: the
    library's stream can be destroyed before the tensors are freed.)"""

    def __init__(self, stream_ptr: int | None, device, tensors, cache: dict | None = None):
        import torch

        self.dev = torch.device(device)
        self.tensors = tensors
        self.cur = torch.cuda.current_stream(self.dev)
        # the handle already on torch's current stream (bench.py, set_stream): stream order
        # is the order of the calls, nothing to add (and nothing to pay per call)
        self.same = bool(stream_ptr) and self.cur.cuda_stream == stream_ptr
        self.lib = None
        if stream_ptr and not self.same:
            key = (stream_ptr, self.dev.index)
            if cache is not None and key in cache:
                self.lib = cache[key]
            else:
                self.lib = torch.cuda.ExternalStream(stream_ptr, device=self.dev)
                if cache is not None:
                    cache.clear()
                    cache[key] = self.lib

    def __enter__(self):
        if self.same:
            return self
        if self.lib is None:  # the call creates its own stream and syncs: order the inputs before it
            self.cur.synchronize()
        else:
            self.lib.wait_stream(self.cur)
        return self

    def __exit__(self, *exc):
        if self.lib is not None:
            self.cur.wait_stream(self.lib)
        return False


def partition_pairs(n_pairs: int, nranks: int, rank: int, far_pairs: float = 0.0) -> tuple[int, int]:
    """The library's multi-GPU split (host only): this rank's [lo, hi) range of
    the near-field (offset, target) pairs in offset-major order; rank 0, which
    also runs the far field, takes round(far_pairs) fewer."""
    lo, hi = C.c_longlong(), C.c_longlong()
    _raise(_native.cuda().fpbem_cu_partition_pairs(int(n_pairs), int(nranks), int(rank), float(far_pairs),
                                                   C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def near_pairs(counts, near_offsets):
    """(offset slot, target cell, source cell) of every near-field pair in the
    library's order: offsets in order, targets x-fastest (BlockToeplitzMatrix
    matvec terms, src/assembly.cpp:62-84)."""
    m = counts
    out = []
    for s, (ox, oy, oz) in enumerate(np.asarray(near_offsets).reshape(-1, 3)):
        for tz in range(m[2]):
            for ty in range(m[1]):
                for tx in range(m[0]):
                    sx, sy, sz = tx - ox, ty - oy, tz - oz
                    if 0 <= sx < m[0] and 0 <= sy < m[1] and 0 <= sz < m[2]:
                        out.append((s, tx + m[0] * (ty + m[1] * tz), sx + m[0] * (sy + m[1] * sz)))
    return out


class Communicator:
    """NCCL communicator of the library (one process per GPU). The 128-byte
    unique id travels over an initialised torch.distributed process group."""

    def __init__(self, device: int, group=None):
        import torch.distributed as dist

        lib = _native.cuda()
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        uid = C.create_string_buffer(128)
        if rank == 0:
            _raise(lib.fpbem_cu_comm_unique_id(uid))
        box = [uid.raw if rank == 0 else None]
        dist.broadcast_object_list(box, src=0, group=group)
        uid = C.create_string_buffer(box[0], 128)
        h = C.c_void_p()
        _raise(lib.fpbem_cu_comm_init(uid, world, rank, device, C.byref(h)))
        self.handle, self.rank, self.nranks = h, rank, world

    def close(self) -> None:
        if getattr(self, "handle", None):
            _native.cuda().fpbem_cu_comm_destroy(self.handle)
            self.handle = None


class HostCommunicator(Communicator):
    """The library's communicator over a torch.distributed process group's
    host all-reduce (gloo): device data is staged through pinned host memory
    (fpbem_cu_comm_from_callback). For ranks without an NCCL path between them
    and for multi-rank tests; the NCCL Communicator is the fast path."""

    def __init__(self, device: int, group=None):
        import torch
        import torch.distributed as dist

        lib = _native.cuda()
        rank, world = dist.get_rank(group), dist.get_world_size(group)

        def allreduce(_ctx, buf, count):
            try:
                arr = np.ctypeslib.as_array(buf, shape=(int(count),))
                dist.all_reduce(torch.from_numpy(arr), group=group)  # in place on the staged host buffer
                return 0
            except Exception:  # noqa: BLE001 - reported to the library as a failed collective
                return 1

        self._cb = _native.ALLREDUCE_FN(allreduce)  # kept alive with the communicator
        h = C.c_void_p()
        _raise(lib.fpbem_cu_comm_from_callback(self._cb, None, world, rank, device, C.byref(h)))
        self.handle, self.rank, self.nranks = h, rank, world


class SimulatedCommunicator(Communicator):
    """Rank `rank` of `nranks` alone on one device (fpbem_cu_comm_simulated):
    collectives move only this rank's own blocks and count the bytes the real
    exchange would send. For timing one rank's share of a multi-GPU product on
    one GPU (tools/model_scaling.py); its products are partial, never answers."""

    def __init__(self, device: int, nranks: int, rank: int):
        h = C.c_void_p()
        _raise(_native.cuda().fpbem_cu_comm_simulated(nranks, rank, device, C.byref(h)))
        self.handle, self.rank, self.nranks = h, rank, nranks

    def traffic(self, reset: bool = False) -> tuple[int, int]:
        """(bytes this rank would have sent, collectives) since the last reset."""
        b, n = C.c_ulonglong(), C.c_longlong()
        _raise(_native.cuda().fpbem_cu_comm_traffic(self.handle, C.byref(b), C.byref(n), int(reset)))
        return int(b.value), int(n.value)


@dataclass
class SolveReport:
    """include/fpbem/solver.hpp:14-19"""

    solution: object
    residual_history: list = field(default_factory=list)
    iterations: int = 0
    converged: bool = False


class FmmOperators:
    """Device-resident periodic single-level FMM operator.

    data: an FmmData (host.Scene.assemble_fmm) or any object with the same
    fields (counts, n_dof, n_coef, near_offsets, near_blocks, far_offsets,
    far_blocks, u0, v0). The spectrum is built on the GPU from the far bank
    unless `lambda_` (reference layout) is given. near_path: "auto" (cost
    model), "direct" (one GEMM per stored offset, BlockToeplitzMatrix::matvec's
    structure) or "lattice" (circulant embedding of the near blocks, one block
    product per Fourier mode).
    """

    NEAR_PATHS = {"auto": 0, "direct": 1, "lattice": 2}

    def __init__(self, data, device: int = 0, fft_sizes=None, lambda_=None, max_rhs: int = 1, lambda_hat=None,
                 near_blocks=None, hat_blocks=None, far_blocks=None, far_hat_blocks=None, near_path: str = "auto",
                 use_symmetries: bool = True):
        lib = _native.cuda()
        self.counts = tuple(int(c) for c in data.counts)
        self.n_dof = int(data.n_dof)
        self.n_coef = int(data.n_coef)
        self.device = device
        self.max_rhs = max_rhs
        n_cells = self.counts[0] * self.counts[1] * self.counts[2]
        self.N = n_cells * self.n_dof
        keep = []

        def ptr(a, dtype):
            a = np.ascontiguousarray(a, dtype=dtype)
            keep.append(a)
            return a.ctypes.data if a.size else None

        d = _native.FmmDesc()
        d.counts[:] = self.counts
        d.n_dof = self.n_dof
        d.n_coef = self.n_coef
        d.n_near = int(len(data.near_offsets))
        d.near_offsets = ptr(data.near_offsets, np.int32)
        on_device = near_blocks is not None
        if on_device:  # CUDA tensors, e.g. from assemble_near_gpu
            keep.append(near_blocks)
            d.near_blocks = near_blocks.data_ptr()
            d.blocks_on_device = 1
        else:
            d.near_blocks = ptr(data.near_blocks, np.complex128)
        d.u0 = ptr(data.u0, np.complex128)
        d.v0 = ptr(data.v0, np.complex128)
        d.fft_sizes[:] = tuple(fft_sizes) if fft_sizes is not None else (0, 0, 0)
        d.lambda_ = ptr(lambda_, np.complex128) if lambda_ is not None else None
        d.n_far = int(len(data.far_offsets))
        d.far_offsets = ptr(data.far_offsets, np.int32)
        if far_blocks is not None:  # CUDA tensors, e.g. from assemble_far_gpu
            keep.append(far_blocks)
            d.far_blocks = far_blocks.data_ptr() if d.n_far else None
            d.far_on_device = 1
        else:
            d.far_blocks = ptr(data.far_blocks, np.complex128)
        level = int(getattr(data, "mirrored_level", -1))
        d.mirrored_level = level
        d.max_rhs = max_rhs
        d.near_path = self.NEAR_PATHS[near_path]
        syms = getattr(data, "cell_symmetries", None) or []  # Scene.cell_symmetries(): mode orbits (extension)
        if syms and use_symmetries:
            d.n_sym = len(syms)
            d.sym_axes = ptr(np.array([g for g, _ in syms], np.int32), np.int32)
            d.sym_perms = ptr(np.stack([np.asarray(p, np.int32) for _, p in syms]), np.int32)
        if level >= 0:
            d.n_hat = int(len(data.hat_indices))
            d.hat_indices = ptr(data.hat_indices, np.int32)
            if on_device:
                keep.append(hat_blocks)
                d.hat_blocks = hat_blocks.data_ptr() if hat_blocks is not None and d.n_hat else None
            else:
                d.hat_blocks = ptr(data.hat_blocks, np.complex128)
            d.n_far_hat = int(len(data.far_hat_indices))
            d.far_hat_indices = ptr(data.far_hat_indices, np.int32)
            if far_blocks is not None:
                keep.append(far_hat_blocks)
                d.far_hat_blocks = far_hat_blocks.data_ptr() if far_hat_blocks is not None and d.n_far_hat else None
            else:
                d.far_hat_blocks = ptr(data.far_hat_blocks, np.complex128)
            d.lambda_hat = ptr(lambda_hat, np.complex128) if lambda_hat is not None else None
        h = C.c_void_p()
        _raise(lib.fpbem_cu_fmm_create(C.byref(d), device, C.byref(h)))
        self._h = h

    def close(self) -> None:
        h = getattr(self, "_h", None)
        if h:
            _native.cuda().fpbem_cu_fmm_destroy(h)
            self._h = None

    def __del__(self):
        self.close()

    @property
    def handle(self):
        return self._h

    def stored_bytes(self) -> int:
        """FmmOperators::stored_bytes (src/fmm.cpp:273-279)."""
        b = C.c_size_t()
        _raise(_native.cuda().fpbem_cu_fmm_bytes(self._h, C.byref(b)))
        return int(b.value)

    def near_path(self) -> tuple[str, tuple[int, int, int], int, int, int, float]:
        """(path, lattice sizes, stored spectrum bytes, Fourier modes per stored
        block (1 without verified symmetries), verified symmetry mask (bit g),
        largest measured symmetry deviation / max|S| or -1) of the near field."""
        p, sizes, nb, mpb, mask, dev = (C.c_int(), (C.c_int * 3)(), C.c_size_t(), C.c_int(), C.c_int(),
                                        C.c_double())
        _raise(_native.cuda().fpbem_cu_fmm_near_path(self._h, C.byref(p), sizes, C.byref(nb), C.byref(mpb),
                                                     C.byref(mask), C.byref(dev)))
        return ({1: "direct", 2: "lattice"}[p.value], tuple(sizes), int(nb.value), mpb.value, mask.value,
                dev.value)

    def spectrum(self) -> tuple[tuple[int, int, int], np.ndarray]:
        sizes = (C.c_int * 3)()
        _raise(_native.cuda().fpbem_cu_spectrum(self._h, sizes, None))
        q = sizes[0] * sizes[1] * sizes[2]
        lam = np.zeros(q * self.n_coef * self.n_coef, np.complex128)
        _raise(_native.cuda().fpbem_cu_spectrum(self._h, sizes, lam.ctypes.data))
        return tuple(sizes), lam

    def far_info(self) -> tuple[tuple[int, int, int], bool]:
        """(M2L lattice sizes, mirror-paired Λ stream)"""
        sizes, paired = (C.c_int * 3)(), C.c_int()
        _raise(_native.cuda().fpbem_cu_far_info(self._h, sizes, C.byref(paired)))
        return tuple(sizes), bool(paired.value)

    def far_parity(self) -> int:
        """0: no parity of Λ; 1: Λ(-q) = D Λ(q) D (a streamed block serves a mode and its mirror);
        2: also Λ(qx, qy, -qz) = Dz Λ(q) Dz (the flat stream reads a quarter of Λ)"""
        sizes, paired = (C.c_int * 3)(), C.c_int()
        _raise(_native.cuda().fpbem_cu_far_info(self._h, sizes, C.byref(paired)))
        return int(paired.value)

    def set_stream(self, stream_ptr: int | None) -> None:
        _raise(_native.cuda().fpbem_cu_set_stream(self._h, stream_ptr))

    def set_partition(self, rank: int, nranks: int, far_pairs: float = 0.0) -> None:
        """Near-field pair partition without communication: matvec returns
        this rank's partial product (rank 0 includes the far field and takes
        round(far_pairs) fewer pairs; every rank must pass the same value)."""
        _raise(_native.cuda().fpbem_cu_fmm_set_partition(self._h, rank, nranks, float(far_pairs)))

    def partition(self) -> tuple[int, int, float]:
        """(lo, hi, far_pairs): this handle's pair range and rank-0 deficit."""
        lo, hi, f = C.c_longlong(), C.c_longlong(), C.c_double()
        _raise(_native.cuda().fpbem_cu_fmm_partition(self._h, C.byref(lo), C.byref(hi), C.byref(f)))
        return lo.value, hi.value, f.value

    def far_pairs(self) -> float:
        """The far field's cost in near-field pair equivalents, measured on
        this device (what set_comm balances rank 0 by)."""
        f = C.c_double()
        _raise(_native.cuda().fpbem_cu_fmm_far_pairs(self._h, C.byref(f)))
        return f.value

    def set_comm(self, comm) -> None:
        """Attach a Communicator: near-field pairs split across its ranks,
        partial products all-reduced over NCCL inside every matvec."""
        _raise(_native.cuda().fpbem_cu_fmm_set_comm(self._h, comm.handle if comm is not None else None))
        self._comm = comm

    def set_slabs(self, comm=None) -> None:
        """Slab-distributed product (lattice near field): this rank owns whole
        planes of cells along the slab axis; matvec_slab maps x[lo:hi) to
        (A x)[lo:hi) with one all-to-all per direction inside, and
        gmres_distributed runs on the slabs. Collective over comm's ranks."""
        _raise(_native.cuda().fpbem_cu_fmm_set_slabs(self._h, comm.handle if comm is not None else None))
        self._slab_comm = comm

    def slab_rows(self) -> tuple[int, int]:
        lo, hi = C.c_longlong(), C.c_longlong()
        _raise(_native.cuda().fpbem_cu_fmm_slab_rows(self._h, C.byref(lo), C.byref(hi)))
        return lo.value, hi.value

    def slab_info(self) -> dict:
        """This rank's slab plan: planes, stored near-field blocks, near and far modes."""
        v = (C.c_longlong * 8)()
        _raise(_native.cuda().fpbem_cu_fmm_slab_info(self._h, v))
        keys = ("rank", "ranks", "axis", "planes", "near_blocks", "near_modes", "far_modes", "z_fused")
        return {k: int(v[i]) for i, k in enumerate(keys)}

    def matvec_slab(self, p):
        """(A x)[lo:hi) from x[lo:hi) (numpy, or a CUDA complex128 tensor)."""
        lo, hi = self.slab_rows()
        lib = _native.cuda()
        if _is_torch(p):
            import torch

            x = p.contiguous()
            if x.numel() != hi - lo or x.dtype != torch.complex128:
                raise ValueError("matvec_slab: expected this rank's rows as complex128")
            y = torch.empty_like(x)
            with self._ordered(x, y):
                _raise(lib.fpbem_cu_fmm_apply_slab(self._h, x.data_ptr(), y.data_ptr(), PTR_DEVICE))
            return y
        x = np.ascontiguousarray(p, dtype=np.complex128)
        if x.size != hi - lo:
            raise ValueError("matvec_slab: expected this rank's rows")
        y = np.empty_like(x)
        _raise(lib.fpbem_cu_fmm_apply_slab(self._h, x.ctypes.data, y.ctypes.data, PTR_HOST))
        return y

    def kernel_launches(self) -> int:
        return int(_native.cuda().fpbem_cu_kernel_launches(self._h))

    def enable_stage_timing(self, on: bool = True, serial: bool = False) -> None:
        """Per-stage CUDA-event timing; serial=True runs P2M + M2L on the main
        stream while timing so every stage is timed alone."""
        _raise(_native.cuda().fpbem_cu_enable_stage_timing(self._h, (2 if serial else 1) if on else 0))

    def stage_times(self) -> dict:
        ms = (C.c_double * 7)()
        _raise(_native.cuda().fpbem_cu_stage_times(self._h, ms))
        keys = ("near_gemm", "near_reduce_l2p", "p2m", "m2l", "total")  # near_gemm: the whole near-field stage
        out = {k: ms[i] for i, k in enumerate(keys)}
        out["applies"] = int(ms[5])
        out["near_mode_product"] = ms[6]
        return out

    def stream_ptr(self) -> int:
        """The cudaStream_t this handle's device work runs on."""
        st = C.c_void_p()
        _raise(_native.cuda().fpbem_cu_get_stream(self._h, C.byref(st)))
        return int(st.value or 0)

    def _ordered(self, *tensors):
        if not hasattr(self, "_stream_cache"):
            self._stream_cache = {}
        return _TorchOrdered(self.stream_ptr(), tensors[0].device, tensors, self._stream_cache)

    def _nrhs(self, p) -> int:
        size = int(p.numel()) if _is_torch(p) else int(np.asarray(p).size)
        if size == 0 or size % self.N:
            raise ValueError("fmm matvec: dimension mismatch")
        return size // self.N

    def matvec(self, p):
        """y = (S + U0 IFFT(Λ FFT(pad(V0 p)))) p. Accepts a host numpy array
        (copied in and out inside the call) or a CUDA torch tensor (device-
        resident, stream-ordered on the handle's stream). Several right-hand
        sides may be stacked one after another."""
        nrhs = self._nrhs(p)
        lib = _native.cuda()
        if _is_torch(p):
            import torch

            if not p.is_cuda or p.dtype != torch.complex128:
                raise ValueError("fmm matvec: expected a complex128 CUDA tensor")
            x = p.contiguous()
            y = torch.empty_like(x)
            with self._ordered(x, y):
                _raise(lib.fpbem_cu_fmm_apply(self._h, x.data_ptr(), y.data_ptr(), nrhs, PTR_DEVICE))
            return y
        x = np.ascontiguousarray(p, dtype=np.complex128)
        y = np.empty_like(x)
        _raise(lib.fpbem_cu_fmm_apply(self._h, x.ctypes.data, y.ctypes.data, nrhs, PTR_HOST))
        return y

    __call__ = matvec


def gmres(apply, b, tol: float = 1e-4, restart: int = 100, max_iter: int = 1000, preconditioner=None,
          device: int = 0):
    """Restarted GMRES from x0 = 0 on the device (src/solver.cpp:21-123).

    apply: an FmmOperators (device-resident Krylov loop, several stacked right-
    hand sides solved independently), or a callable mapping a CUDA complex128
    torch tensor to a new one (the ApplyFn seam, include/fpbem/solver.hpp:21).
    Returns a SolveReport, or a list of them for stacked right-hand sides.
    """
    lib = _native.cuda()
    is_t = _is_torch(b)
    if isinstance(apply, FmmOperators):
        nrhs = apply._nrhs(b)
        its = (C.c_int * nrhs)()
        conv = (C.c_int * nrhs)()
        cap = max(1, max_iter)
        hist = np.zeros(nrhs * cap)
        hlen = (C.c_int * nrhs)()
        if preconditioner is not None:
            raise ValueError("gmres: preconditioners are supported through the callable form")
        if is_t:
            bx = b.contiguous()
            import torch

            x = torch.empty_like(bx)
            with apply._ordered(bx, x):
                rc = lib.fpbem_cu_gmres(apply.handle, bx.data_ptr(), x.data_ptr(), nrhs, tol, restart, max_iter,
                                        PTR_DEVICE, its, conv, hist.ctypes.data_as(_native.c_double_p), cap, hlen)
        else:
            bx = np.ascontiguousarray(b, np.complex128)
            x = np.zeros_like(bx)
            rc = lib.fpbem_cu_gmres(apply.handle, bx.ctypes.data, x.ctypes.data, nrhs, tol, restart, max_iter,
                                    PTR_HOST, its, conv, hist.ctypes.data_as(_native.c_double_p), cap, hlen)
        _raise(rc)
        n = apply.N
        reps = [SolveReport(x[r * n:(r + 1) * n], list(hist[r * cap:r * cap + hlen[r]]), int(its[r]),
                            bool(conv[r])) for r in range(nrhs)]
        return reps[0] if nrhs == 1 else reps
    return _gmres_callable(apply, b, tol, restart, max_iter, preconditioner, device)


def gmres_distributed(op: FmmOperators, b, tol: float = 1e-4, restart: int = 100, max_iter: int = 1000):
    """Restarted GMRES with the Krylov basis split over the ranks of the
    operator's communicator (FmmOperators.set_comm) in slabs of whole cells
    (SURVEY §8e): per step one all-gather, one reduce-scatter and one batched
    all-reduce per classical Gram-Schmidt pass, with the reference's
    reorthogonalisation test (fpbem_cu_gmres_dist). Every rank passes the full
    right-hand side (numpy or CUDA tensor) and gets the full solution. Without
    a communicator it runs on the operator's device alone."""
    lib = _native.cuda()
    if op._nrhs(b) != 1:
        raise ValueError("gmres_distributed: one right-hand side")
    its, conv, hlen = C.c_int(), C.c_int(), C.c_int()
    cap = max(1, max_iter)
    hist = np.zeros(cap)
    hp = hist.ctypes.data_as(_native.c_double_p)
    if _is_torch(b):
        import torch

        bx = b.contiguous()
        x = torch.empty_like(bx)
        with op._ordered(bx, x):
            rc = lib.fpbem_cu_gmres_dist(op.handle, bx.data_ptr(), x.data_ptr(), tol, restart, max_iter, PTR_DEVICE,
                                         C.byref(its), C.byref(conv), hp, cap, C.byref(hlen))
    else:
        bx = np.ascontiguousarray(b, np.complex128)
        x = np.zeros_like(bx)
        rc = lib.fpbem_cu_gmres_dist(op.handle, bx.ctypes.data, x.ctypes.data, tol, restart, max_iter, PTR_HOST,
                                     C.byref(its), C.byref(conv), hp, cap, C.byref(hlen))
    _raise(rc)
    return SolveReport(x, list(hist[:hlen.value]), its.value, bool(conv.value))


def dist_rows(op: FmmOperators) -> tuple[int, int]:
    """This rank's slab [lo, hi) of the global rows under gmres_distributed."""
    lo, hi = C.c_longlong(), C.c_longlong()
    _raise(_native.cuda().fpbem_cu_gmres_dist_rows(op.handle, C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def rhs_shard(n_rhs: int, world: int, rank: int) -> list[int]:
    """Right-hand sides this rank solves when independent solves are sharded
    (SURVEY §8e, cfg5): round-robin, so ranks differ by at most one solve."""
    if world < 1 or not 0 <= rank < world or n_rhs < 0:
        raise ValueError("rhs_shard: bad world / rank / count")
    return list(range(rank, n_rhs, world))


def gmres_sharded(op, b, n_rhs: int, tol: float = 1e-4, restart: int = 100, max_iter: int = 1000, group=None,
                  solve=None):
    """Independent GMRES solves of n_rhs stacked right-hand sides `b` (numpy,
    every rank holding all of them) sharded over the ranks of a
    torch.distributed group: each rank solves its rhs_shard in one lockstep
    batch (FmmOperators with max_rhs >= its share) and the reports are
    gathered, so every rank returns all n_rhs SolveReports in order. No
    collective inside the solves (the operator is replicated). `solve`
    overrides the per-rank solver (for tests)."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    bb = np.ascontiguousarray(b, np.complex128).reshape(n_rhs, -1)
    mine = rhs_shard(n_rhs, world, rank)
    if solve is None:
        def solve(rhs):
            reps = gmres(op, np.ascontiguousarray(rhs).reshape(-1), tol=tol, restart=restart, max_iter=max_iter)
            return reps if isinstance(reps, list) else [reps]
    local = solve(bb[mine]) if mine else []
    payload = [(i, np.asarray(r.solution), list(r.residual_history), r.iterations, r.converged)
               for i, r in zip(mine, local)]
    gathered = [payload]
    if world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, payload, group=group)
    out = [None] * n_rhs
    for part in gathered:
        for i, sol, hist, its, conv in part:
            out[i] = SolveReport(sol, hist, its, conv)
    return out


def _cell_struct(scene, keep):
    c = scene.cell()
    n = len(c["area"])
    arrs = {
        "corners": np.ascontiguousarray(c["corners"], np.float64),
        "nv": np.ascontiguousarray(c["nv"], np.int32),
        "centroid": np.ascontiguousarray(c["centroid"], np.float64),
        "normal": np.ascontiguousarray(-c["normal"], np.float64),  # BIE orientation (assembly.cpp:17-21)
        "diameter": np.ascontiguousarray(c["diameter"], np.float64),
    }
    keep.append(arrs)
    cs = _native.Cell()
    cs.n = n
    for k, a in arrs.items():
        setattr(cs, k, a.ctypes.data)
    cs.beta = None  # rigid scenes
    return cs, n


def assemble_near_gpu(scene, data, device: int = 0, halfspace=None):
    """Near-field blocks S_o of `data`'s offsets assembled on the GPU
    (fpbem_cu_assemble_near); returns a CUDA complex128 tensor (n_near, n, n)
    holding column-major blocks, ready for FmmOperators(near_blocks=...).
    halfspace=(axis, offset, reflection) folds the image terms (mirror axis
    not periodic)."""
    import torch

    keep = []
    cs, n = _cell_struct(scene, keep)
    k = float(scene.wavenumber)
    alpha = _native.C64(0.0, -1.0 / k)
    pitch = np.ascontiguousarray(scene.pitch, np.float64)
    offs = np.ascontiguousarray(data.near_offsets, np.int32)
    out = torch.empty((len(offs), n, n), dtype=torch.complex128, device=f"cuda:{device}")
    fold, axis, off, refl = 0, 2, 0.0, 0j
    if halfspace is not None:
        fold = 1
        axis, off, refl = halfspace
    rc = _native.cuda().fpbem_cu_assemble_near(C.byref(cs), k, alpha, pitch.ctypes.data_as(_native.c_double_p),
                                               len(offs), offs.ctypes.data_as(_native.c_int_p), fold, int(axis),
                                               float(off), _native.C64(complex(refl).real, complex(refl).imag),
                                               device, out.data_ptr(), PTR_DEVICE)
    _raise(rc)
    return out


def assemble_hat_gpu(scene, data, halfspace, device: int = 0):
    """S_hat blocks of a split half space on the GPU (fpbem_cu_assemble_hat)."""
    import torch

    keep = []
    cs, n = _cell_struct(scene, keep)
    k = float(scene.wavenumber)
    pitch = np.ascontiguousarray(scene.pitch, np.float64)
    counts = np.ascontiguousarray(data.counts, np.int32)
    idx = np.ascontiguousarray(data.hat_indices, np.int32)
    out = torch.empty((max(len(idx), 1), n, n), dtype=torch.complex128, device=f"cuda:{device}")
    axis, off, refl = halfspace
    rc = _native.cuda().fpbem_cu_assemble_hat(C.byref(cs), k, _native.C64(0.0, -1.0 / k),
                                              pitch.ctypes.data_as(_native.c_double_p),
                                              counts.ctypes.data_as(_native.c_int_p), len(idx),
                                              idx.ctypes.data_as(_native.c_int_p), int(axis), float(off),
                                              _native.C64(complex(refl).real, complex(refl).imag), device,
                                              out.data_ptr(), PTR_DEVICE)
    _raise(rc)
    return out[: len(idx)]


def m2l_bank_gpu(n_t: int, k: float, delta=None, image_delta=None, parity_axis: int = 2, reflection=0.0,
                 device: int = 0):
    """K blocks on the GPU (fpbem_cu_m2l_bank): for each row s of the (n, 3)
    translation vectors, K(delta_s) [+ reflection K(image_delta_s) P_axis].
    Returns a CUDA complex128 tensor (n, b, b) of column-major b x b blocks
    (index [s, col, row]), b = (n_t + 1)^2 — TranslationTable::m2l
    (src/specfun.cpp:332-351) for many offsets at once."""
    import torch

    dl = None if delta is None else np.ascontiguousarray(delta, np.float64).reshape(-1, 3)
    im = None if image_delta is None else np.ascontiguousarray(image_delta, np.float64).reshape(-1, 3)
    n = len(dl) if dl is not None else (len(im) if im is not None else 0)
    if dl is not None and im is not None and len(im) != n:
        raise ValueError("m2l_bank_gpu: delta and image_delta lengths differ")
    b = (n_t + 1) ** 2
    out = torch.empty((max(n, 1), b, b), dtype=torch.complex128, device=f"cuda:{device}")
    r = complex(reflection)
    _raise(_native.cuda().fpbem_cu_m2l_bank(
        int(n_t), float(k), n, dl.ctypes.data_as(_native.c_double_p) if dl is not None else None,
        im.ctypes.data_as(_native.c_double_p) if im is not None else None, int(parity_axis),
        _native.C64(r.real, r.imag), device, out.data_ptr(), PTR_DEVICE))
    return out[:n]


def far_translation_vectors(scene, data, halfspace=None):
    """Translation vectors of the far K bank of `data`, as assemble_periodic_fmm
    uses them (src/fmm.cpp:180-191, 204-242): returns (delta, image_delta,
    hat_image_delta); image terms only for a half space (axis, offset,
    reflection) — folded when data.mirrored_level < 0, split otherwise."""
    pitch = np.asarray(scene.pitch, np.float64)
    _, _, base, _ = scene.classify()
    offs = np.asarray(data.far_offsets, np.float64).reshape(-1, 3)
    delta = offs * pitch
    image = hat = None
    if halfspace is not None:
        axis, off, _ = halfspace
        mirror = base.copy()
        mirror[axis] = 2.0 * off - base[axis]
        level = int(getattr(data, "mirrored_level", -1))
        if level < 0:  # folded: center(o) - mirror(base_center)
            image = base + delta - mirror
        else:  # split: target_center - image_center over the far Hankel indices
            idx = np.asarray(data.far_hat_indices, np.int64).reshape(-1, 3)
            m = np.asarray(data.counts, np.int64)
            tgt = idx.copy()
            tgt[:, axis] = np.minimum(idx[:, axis], m[axis] - 1)
            src = np.zeros_like(idx)
            src[:, axis] = idx[:, axis] - tgt[:, axis]
            sshift = src * pitch
            sshift[:, axis] = -sshift[:, axis]
            hat = (base + tgt * pitch) - (mirror + sshift)
    return delta, image, hat


def assemble_far_gpu(scene, data, n_t: int = 4, halfspace=None, device: int = 0):
    """K bank (and K_hat bank of a split half space) of `data` on the GPU:
    returns (far_blocks, far_hat_blocks or None) as CUDA tensors for
    FmmOperators(far_blocks=..., far_hat_blocks=...). `data` may come from
    Scene.assemble_fmm(..., skip_far_values=True)."""
    k = float(scene.wavenumber)
    delta, image, hat = far_translation_vectors(scene, data, halfspace)
    refl = complex(halfspace[2]) if halfspace is not None else 0.0
    axis = int(halfspace[0]) if halfspace is not None else 2
    far = m2l_bank_gpu(n_t, k, delta, image, axis, refl, device)
    far_hat = m2l_bank_gpu(n_t, k, None, hat, axis, refl, device) if hat is not None else None
    return far, far_hat


def evaluate_field_gpu(scene, solution, points, field: int = 0, p_incident=None, device: int = 0):
    """Pressure at observation points (postproc::evaluate_field,
    src/postproc.cpp:39-62) on the GPU: p_inc (host incident field of `field`,
    with the scene's half-space images, unless given) + the representation
    formula over the replicated mesh and, with a half space, its mirror image.
    solution: numpy array (host) or CUDA tensor; returns the same kind."""
    import torch

    keep = []
    cs, n = _cell_struct(scene, keep)
    pts = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
    pitch = np.ascontiguousarray(scene.pitch, np.float64)
    counts = np.ascontiguousarray(scene.counts, np.int32)
    hs = getattr(scene, "halfspace", None)
    axis, off, refl = hs if hs is not None else (2, 0.0, 0j)
    if p_incident is None:
        p_incident = scene.incident(pts, field)
    lib = _native.cuda()
    if _is_torch(solution):
        sol = solution.to(torch.complex128).contiguous()
        pinc = (p_incident if _is_torch(p_incident) else torch.from_numpy(np.asarray(p_incident, np.complex128))).to(
            sol.device).contiguous()
        out = torch.empty(len(pts), dtype=torch.complex128, device=sol.device)
        args = (sol.data_ptr(), pinc.data_ptr(), out.data_ptr(), PTR_DEVICE, sol.device.index)
    else:
        sol = np.ascontiguousarray(solution, np.complex128)
        pinc = np.ascontiguousarray(p_incident, np.complex128)
        out = np.zeros(len(pts), np.complex128)
        args = (sol.ctypes.data, pinc.ctypes.data, out.ctypes.data, PTR_HOST, device)

    def call():
        _raise(lib.fpbem_cu_evaluate_field(C.byref(cs), float(scene.wavenumber),
                                           pitch.ctypes.data_as(_native.c_double_p),
                                           counts.ctypes.data_as(_native.c_int_p), args[0], len(pts),
                                           pts.ctypes.data_as(_native.c_double_p), args[1], int(axis), float(off),
                                           _native.C64(complex(refl).real, complex(refl).imag), args[4], args[2],
                                           args[3]))

    if _is_torch(solution):
        with _TorchOrdered(None, sol.device, (sol, pinc, out)):  # the call syncs its own stream
            call()
    else:
        call()
    return out


def _gmres_callable(apply, b, tol, restart, max_iter, preconditioner, device):
    import torch

    lib = _native.cuda()
    dev = torch.device("cuda", device)
    bt = (b if _is_torch(b) else torch.from_numpy(np.ascontiguousarray(b, np.complex128))).to(dev).contiguous()
    n = bt.numel()
    errors: list[BaseException] = []

    def wrap(fn):
        def cb(_ctx, x_ptr, y_ptr, stream_ptr):
            try:
                with torch.cuda.stream(torch.cuda.ExternalStream(stream_ptr, device=dev)):
                    xin = _from_ptr(x_ptr, n, dev)
                    out = fn(xin.clone())
                    _from_ptr(y_ptr, n, dev).copy_(out.reshape(-1))
                return 0
            except BaseException as e:  # reported through the C return code
                errors.append(e)
                return 1

        return _native.APPLY_FN(cb)

    acb = wrap(apply)
    pcb = wrap(preconditioner) if preconditioner is not None else _native.APPLY_FN()
    x = torch.empty_like(bt)
    its, conv, hlen = C.c_int(), C.c_int(), C.c_int()
    cap = max(1, max_iter)
    hist = np.zeros(cap)
    torch.cuda.synchronize(dev)
    rc = lib.fpbem_cu_gmres_fn(device, n, acb, None, pcb, None, bt.data_ptr(), x.data_ptr(), tol, restart,
                               max_iter, PTR_DEVICE, C.byref(its), C.byref(conv),
                               hist.ctypes.data_as(_native.c_double_p), cap, C.byref(hlen))
    if errors and rc != ENONFINITE:
        raise errors[0]
    _raise(rc)
    sol = x if _is_torch(b) else x.cpu().numpy()
    return SolveReport(sol, list(hist[: hlen.value]), its.value, bool(conv.value))


def _from_ptr(ptr: int, n: int, dev):
    """Wrap a raw device pointer of n complex128 values as a torch tensor (no copy)."""
    import torch

    class _Holder:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<c16", "data": (int(ptr), False), "version": 3,
                                    "strides": None}

    return torch.as_tensor(_Holder(), device=dev)
