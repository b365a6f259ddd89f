"""GPU parity: the sm_100a path through the C-ABI against the CPU oracle on
identical seeded inputs. Tolerances from BASELINE.json's north_star: matvec
relative L2 <= 1e-10 (fp64 complex), GMRES iterations equal within +-1 and
solutions within 1e-8 relative."""
import numpy as np
import pytest

import oracle as O
from conftest import rel

pytestmark = pytest.mark.gpu

MATVEC_TOL = 1e-10
SOLVE_TOL = 1e-8


class Data:
    """FmmData-like bundle for synthetic operators."""

    def __init__(self, counts, n, b, near_offsets, near_blocks, far_offsets, far_blocks, u0, v0):
        self.counts, self.n_dof, self.n_coef = tuple(counts), n, b
        self.near_offsets = np.asarray(near_offsets, np.int32).reshape(-1, 3)
        self.near_blocks = np.asarray(near_blocks, np.complex128)
        self.far_offsets = np.asarray(far_offsets, np.int32).reshape(-1, 3)
        self.far_blocks = np.asarray(far_blocks, np.complex128)
        self.u0, self.v0 = np.asarray(u0, np.complex128), np.asarray(v0, np.complex128)

    @property
    def N(self):
        return int(np.prod(self.counts)) * self.n_dof


def all_offsets(counts):
    return [(x, y, z) for z in range(1 - counts[2], counts[2]) for y in range(1 - counts[1], counts[1])
            for x in range(1 - counts[0], counts[0])]


def crand(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def uvec(rng, n):  # BASELINE inputs: re/im i.i.d. U[-1, 1]
    return rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)


def toeplitz_only(rng, counts, n, b=4):
    """near field = full random Toeplitz; expansions zero -> y = S p"""
    offs = all_offsets(counts)
    return Data(counts, n, b, offs, crand(rng, len(offs), n, n), np.zeros((0, 3)), np.zeros((0, b, b)),
                np.zeros((b, n)), np.zeros((n, b)))


def circulant_only(rng, counts, b):
    """K = full random Toeplitz of b x b blocks, V0 = U0 = I, S = 0 -> y = K p"""
    offs = all_offsets(counts)
    eye = np.eye(b, dtype=np.complex128)
    return Data(counts, b, b, [(0, 0, 0)], np.zeros((1, b, b)), offs, crand(rng, len(offs), b, b), eye, eye)


@pytest.fixture(scope="module")
def ops():
    from paper_2201_12050_b200 import FmmOperators

    return FmmOperators


@pytest.mark.parametrize("counts", [(1, 1, 1), (2, 1, 1), (3, 3, 1), (5, 1, 2), (2, 3, 2), (1, 16, 1)])
@pytest.mark.parametrize("n", [3, 24, 70, 130])
def test_near_field_toeplitz_matches_oracle_and_dense(ops, counts, n):
    rng = np.random.default_rng(n + 7 * counts[0] + 11 * counts[1] + 13 * counts[2])
    d = toeplitz_only(rng, counts, n)
    op = ops(d)
    p = uvec(rng, d.N)
    ref = O.toeplitz_matvec(counts, d.near_offsets, d.near_blocks, p)
    assert rel(op.matvec(p), ref) <= MATVEC_TOL
    if d.N <= 600:
        dense = O.toeplitz_expand_dense(counts, d.near_offsets, d.near_blocks)
        assert rel(op.matvec(p), dense @ p) <= MATVEC_TOL


def test_near_field_banded_offset_subset(ops):
    """near field with a subset of offsets (absent offsets act as zero blocks)"""
    rng = np.random.default_rng(3)
    counts, n = (4, 5, 3), 40
    offs = [o for o in all_offsets(counts) if abs(o[0]) + abs(o[1]) + abs(o[2]) <= 2]
    d = toeplitz_only(rng, counts, n)
    d.near_offsets = np.asarray(offs, np.int32)
    d.near_blocks = crand(rng, len(offs), n, n)
    p = uvec(rng, d.N)
    assert rel(ops(d).matvec(p), O.toeplitz_matvec(counts, offs, d.near_blocks, p)) <= MATVEC_TOL


@pytest.mark.parametrize("counts", [(2, 1, 1), (3, 1, 1), (5, 3, 1), (1, 16, 1), (3, 3, 2), (4, 4, 4), (8, 1, 1)])
@pytest.mark.parametrize("b", [1, 3, 25])
def test_circulant_m2l_matches_oracle(ops, counts, b):
    """CirculantSpectrum::matvec (src/structured.cpp:122-166) on the device,
    incl. 7-smooth padded lengths (2M-1 = 31 -> 32) and single-cell axes."""
    rng = np.random.default_rng(b * 100 + sum(counts))
    d = circulant_only(rng, counts, b)
    op = ops(d)
    p = uvec(rng, d.N)
    sizes, lam = O.spectrum_build(counts, d.far_offsets, d.far_blocks)
    gsizes, glam = op.spectrum()
    assert gsizes == sizes
    assert rel(glam, lam) <= 1e-12
    ref = O.spectrum_matvec(counts, sizes, b, lam, p)
    assert rel(op.matvec(p), ref) <= MATVEC_TOL
    if d.N <= 400:
        dense = O.toeplitz_expand_dense(counts, d.far_offsets, d.far_blocks)
        assert rel(op.matvec(p), dense @ p) <= MATVEC_TOL


@pytest.mark.parametrize("zmode", ["fused", "stream"])
@pytest.mark.parametrize("counts,b", [((3, 3, 2), 25), ((4, 4, 4), 9), ((2, 3, 5), 25), ((1, 4, 3), 4), ((6, 5, 9), 16)])
def test_m2l_z_forms_match_oracle(ops, monkeypatch, counts, b, zmode):
    """The two forms of the far field's z stage — the fused per-column kernel and the z axis passes
    around the flat Λ stream (the default; FPBEM_M2L_Z=fused selects the other) — both equal CirculantSpectrum::matvec
    (src/structured.cpp:122-166); random blocks have no mirror parity, so every column is its own item."""
    monkeypatch.setenv("FPBEM_M2L_Z", zmode)
    rng = np.random.default_rng(b + sum(counts))
    d = circulant_only(rng, counts, b)
    op = ops(d)
    p = uvec(rng, d.N)
    ref = O.toeplitz_matvec(counts, d.far_offsets, d.far_blocks, p)
    y = op.matvec(p)
    assert rel(y, ref) <= MATVEC_TOL
    assert np.array_equal(y, op.matvec(p))


@pytest.mark.parametrize("zmode", ["fused", "stream"])
def test_m2l_z_forms_many_modes_per_cta(ops, monkeypatch, zmode):
    """32 x 32 x 8 modes: every CTA of the persistent kernels takes several times its ring of Λ blocks,
    so the ring slots wrap and their mbarrier phases are reused (bitwise repeatable, = the oracle's
    FFT-based CirculantSpectrum::matvec)."""
    monkeypatch.setenv("FPBEM_M2L_Z", zmode)
    rng = np.random.default_rng(99)
    counts, b = (16, 16, 4), 25
    d = circulant_only(rng, counts, b)
    op = ops(d)
    p = uvec(rng, d.N)
    sizes, lam = O.spectrum_build(counts, d.far_offsets, d.far_blocks)
    ref = O.spectrum_matvec(counts, sizes, b, lam, p)
    y = op.matvec(p)
    assert rel(y, ref) <= MATVEC_TOL
    for _ in range(5):
        assert np.array_equal(y, op.matvec(p))


@pytest.mark.parametrize("cid,var", [(3, 2), (5, 2)])
def test_m2l_flat_stream_on_paired_spectrum(ops, assembled, monkeypatch, cid, var):
    """An assembled operator's Λ has the mirror parity Λ(-q) = D Λ(q) D and the reflection parity
    Λ(qx, qy, -qz) = Dz Λ(q) Dz: one streamed block serves a mode and its mirror (two modes per block,
    FPBEM_M2L_QUAD=0) or four modes (the default); both equal the oracle and the fused z kernel,
    2 right-hand sides included (E = 2 b fields per mode)."""
    sc, d = assembled(cid, var)
    ora = O.OracleFmm(d)
    rng = np.random.default_rng(17 + cid)
    P = [uvec(rng, d.N) for _ in range(2)]
    refs = [ora.matvec(p) for p in P]
    monkeypatch.setenv("FPBEM_M2L_Z", "fused")
    y_fused = ops(d).matvec(P[0])
    monkeypatch.setenv("FPBEM_M2L_Z", "stream")
    for quad in ("0", "1"):
        monkeypatch.setenv("FPBEM_M2L_QUAD", quad)
        op = ops(d, max_rhs=2)
        assert op.far_info()[1] and op.far_parity() == 2
        y = op.matvec(np.concatenate(P))
        for r in range(2):
            assert rel(y[r * d.N:(r + 1) * d.N], refs[r]) <= MATVEC_TOL
        assert rel(y[:d.N], y_fused) <= 1e-14
        assert np.array_equal(y, op.matvec(np.concatenate(P)))


@pytest.mark.parametrize("n_t", [2, 3])
def test_m2l_flat_stream_other_orders(ops, monkeypatch, n_t):
    """Expansion orders other than the default n_t = 4 (b = 9, 16: the stream kernel's generic column
    loop, four modes per block) against the oracle and the fused z kernel."""
    from paper_2201_12050_b200 import Scene

    d = Scene(3, 2).assemble_fmm(n_t)
    ora = O.OracleFmm(d)
    p = uvec(np.random.default_rng(n_t), d.N)
    monkeypatch.setenv("FPBEM_M2L_Z", "fused")
    y_fused = ops(d).matvec(p)
    monkeypatch.setenv("FPBEM_M2L_Z", "stream")
    op = ops(d)
    assert op.far_parity() == 2
    y = op.matvec(p)
    assert rel(y, ora.matvec(p)) <= MATVEC_TOL
    assert rel(y, y_fused) <= 1e-14


def test_scalar_toeplitz_known_answer_on_device(ops):
    """test_structured.cpp:84-98 through the device M2L: T=[[2,1],[3,2]], T(1,1)=(3,5)"""
    d = Data((2, 1, 1), 1, 1, [(0, 0, 0)], np.zeros((1, 1, 1)), [(0, 0, 0), (1, 0, 0), (-1, 0, 0)],
             np.array([[[2]], [[3]], [[1]]]), np.eye(1), np.eye(1))
    y = ops(d).matvec(np.array([1, 1], np.complex128))
    np.testing.assert_allclose(y, [3, 5], atol=1e-14)


def test_caller_chosen_fft_sizes(ops):
    """any L >= 2M-1 is exact (SURVEY finding 7)"""
    rng = np.random.default_rng(8)
    counts = (5, 3, 1)
    d = circulant_only(rng, counts, 4)
    p = uvec(rng, d.N)
    ref = O.toeplitz_matvec(counts, d.far_offsets, d.far_blocks, p)
    for sizes in [(9, 5, 1), (16, 8, 1), (10, 7, 1)]:
        assert rel(ops(d, fft_sizes=sizes).matvec(p), ref) <= MATVEC_TOL
    with pytest.raises(ValueError):
        ops(d, fft_sizes=(8, 5, 1))


def test_prebuilt_reference_spectrum_is_accepted(ops):
    rng = np.random.default_rng(12)
    counts = (3, 4, 1)
    d = circulant_only(rng, counts, 5)
    sizes, lam = O.spectrum_build(counts, d.far_offsets, d.far_blocks)
    op = ops(d, fft_sizes=sizes, lambda_=lam)
    p = uvec(rng, d.N)
    assert rel(op.matvec(p), O.spectrum_matvec(counts, sizes, 5, lam, p)) <= MATVEC_TOL


# ---- assembled operators of the BASELINE configurations -----------------------------

SMALL_SCENES = [(1, 0), (1, 1), (2, 2), (3, 2), (4, 2), (5, 2), (6, 8), (6, 16)]


@pytest.fixture(scope="module")
def assembled():
    from paper_2201_12050_b200 import Scene

    cache = {}

    def get(cid, var):
        if (cid, var) not in cache:
            sc = Scene(cid, var)
            cache[(cid, var)] = (sc, sc.assemble_fmm(4))
        return cache[(cid, var)]

    return get


@pytest.mark.parametrize("cid,var", SMALL_SCENES)
def test_fmm_matvec_matches_oracle(ops, assembled, cid, var):
    sc, d = assembled(cid, var)
    ora = O.OracleFmm(d)
    op = ops(d)
    rng = np.random.default_rng(cid)  # seed = config id (BASELINE.md CPU-baseline plan)
    p = uvec(rng, d.N)
    assert rel(op.matvec(p), ora.matvec(p)) <= MATVEC_TOL
    sizes, lam = op.spectrum()
    assert sizes == ora.sizes
    if d.n_far:
        assert rel(lam, ora.lambda_) <= 1e-12
    assert op.stored_bytes() == 16 * (d.n_near * d.n_dof ** 2 + int(np.prod(sizes)) * 625 + 2 * 25 * d.n_dof)


def test_multi_rhs_equals_single_rhs(ops, assembled):
    sc, d = assembled(3, 2)
    rng = np.random.default_rng(5)
    P = [uvec(rng, d.N) for _ in range(3)]
    single = ops(d).matvec
    multi = ops(d, max_rhs=2)  # 3 rhs through chunks of 2
    y = multi.matvec(np.concatenate(P))
    for r in range(3):
        assert rel(y[r * d.N:(r + 1) * d.N], single(P[r])) <= 1e-14


@pytest.mark.parametrize("cid,var,nrhs", [(1, 0, 4), (2, 2, 5), (3, 2, 8), (5, 2, 70), (4, 2, 6), (1, 1, 13)])
def test_multi_rhs_tensor_core_mode_product(ops, assembled, cid, var, nrhs):
    """From 4 right-hand sides the per-mode product is a DMMA contraction
    (mode_gemm_kernel), and the P2M (p2m_gemm_kernel); 70 rhs = two
    row blocks: every rhs equals its own single-rhs product and the oracle."""
    sc, d = assembled(cid, var)
    rng = np.random.default_rng(nrhs)
    P = [uvec(rng, d.N) for _ in range(nrhs)]
    y = ops(d, max_rhs=nrhs).matvec(np.concatenate(P))
    single = ops(d)
    ora = O.OracleFmm(d)
    for r in (0, nrhs // 2, nrhs - 1):
        yr = y[r * d.N:(r + 1) * d.N]
        assert rel(yr, single.matvec(P[r])) <= 1e-13
        assert rel(yr, ora.matvec(P[r])) <= MATVEC_TOL


def test_device_pointer_apply_matches_host_pointer(ops, assembled):
    torch = pytest.importorskip("torch")
    sc, d = assembled(5, 2)
    op = ops(d)
    rng = np.random.default_rng(2)
    p = uvec(rng, d.N)
    yh = op.matvec(p)
    yd = op.matvec(torch.from_numpy(p).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(yd.cpu().numpy(), yh)


@pytest.mark.parametrize("b", [144, 169, 256])
@pytest.mark.parametrize("path", ["direct", "lattice"])
def test_large_expansion_order_matches_oracle(ops, b, path):
    """n_t = 11, 12, 15 (b = (n_t+1)^2 > 128 coefficients, more than one CTA
    of the reduction / L2P kernels loads at once): full FMM product on both
    near-field paths against the oracle."""
    rng = np.random.default_rng(b)
    counts, n = (3, 2, 2), 40
    offs = all_offsets(counts)
    near = [o for o in offs if max(abs(c) for c in o) <= 1]
    far = [o for o in offs if max(abs(c) for c in o) > 1]
    d = Data(counts, n, b, near, crand(rng, len(near), n, n), far, 0.01 * crand(rng, len(far), b, b),
             crand(rng, n, b) / b, crand(rng, b, n) / n)
    p = uvec(rng, d.N)
    assert rel(ops(d, near_path=path).matvec(p), O.OracleFmm(d).matvec(p)) <= MATVEC_TOL


def test_device_pointer_apply_is_ordered_against_torch_stream(ops, assembled):
    """The input is produced on torch's current stream behind a long kernel and
    the output consumed there, with no explicit synchronisation in between:
    the library stream waits for the producer and torch waits for the product."""
    torch = pytest.importorskip("torch")
    sc, d = assembled(3, 2)
    op = ops(d)
    rng = np.random.default_rng(12)
    p = uvec(rng, d.N)
    yh = op.matvec(p)
    big = torch.randn(4096, 4096, device="cuda", dtype=torch.float64)
    for _ in range(3):
        big = big @ big / 64.0  # keeps torch's stream busy for a while
        x = torch.from_numpy(p).cuda(non_blocking=False) * (1.0 + 0.0 * big[0, 0])
        y = op.matvec(x)
        z = (y * 1.0).cpu().numpy()
        assert np.array_equal(z, yh)


def test_apply_is_deterministic_and_linear(ops, assembled):
    sc, d = assembled(2, 2)
    op = ops(d)
    rng = np.random.default_rng(4)
    p, q = uvec(rng, d.N), uvec(rng, d.N)
    y1 = op.matvec(p)
    assert np.array_equal(y1, op.matvec(p))  # fixed-order reductions, no atomics
    a = 0.3 - 1.1j
    assert rel(op.matvec(a * p + q), a * y1 + op.matvec(q)) < 1e-13


def test_dimension_mismatch_raises_invalid_argument(ops, assembled):
    sc, d = assembled(1, 0)
    with pytest.raises(ValueError, match="dimension mismatch"):
        ops(d).matvec(np.zeros(d.N + 1, np.complex128))


# ---- GMRES ------------------------------------------------------------------------

@pytest.mark.parametrize("cid,var", [(1, 0), (3, 2), (4, 2), (5, 2), (6, 8)])
def test_fmm_gmres_matches_oracle(ops, assembled, cid, var):
    from paper_2201_12050_b200 import gmres

    sc, d = assembled(cid, var)
    b = sc.rhs(0)
    rep = gmres(ops(d), b, tol=1e-6, restart=50, max_iter=400)
    x, its, conv, hist = O.OracleFmm(d).gmres(b, tol=1e-6, restart=50, max_iter=400)
    assert rep.converged == conv
    assert abs(rep.iterations - its) <= 1
    assert rel(rep.solution, x) <= SOLVE_TOL
    assert len(rep.residual_history) == rep.iterations


def test_fmm_gmres_with_restarts_matches_oracle(ops, assembled):
    from paper_2201_12050_b200 import gmres

    sc, d = assembled(2, 2)
    b = sc.rhs(0)
    rep = gmres(ops(d), b, tol=1e-6, restart=10, max_iter=2000)
    x, its, conv, hist = O.OracleFmm(d).gmres(b, tol=1e-6, restart=10, max_iter=2000)
    assert rep.converged and conv
    assert abs(rep.iterations - its) <= 1
    assert rel(rep.solution, x) <= SOLVE_TOL
    n = min(len(hist), len(rep.residual_history))
    assert rel(np.array(rep.residual_history[:n]), np.array(hist[:n])) < 1e-8


def test_fmm_gmres_multi_rhs(ops, assembled):
    from paper_2201_12050_b200 import gmres

    sc, d = assembled(5, 2)
    sc.set_sources([1, 1], [[1, 0, 0], [0, 0.6, 0.8]])
    b = np.concatenate([sc.rhs(0), sc.rhs(1)])
    reps = gmres(ops(d), b, tol=1e-6, restart=50, max_iter=400)
    ora = O.OracleFmm(d)
    for r in range(2):
        x, its, conv, _ = ora.gmres(b[r * d.N:(r + 1) * d.N], tol=1e-6, restart=50, max_iter=400)
        assert abs(reps[r].iterations - its) <= 1
        assert rel(reps[r].solution, x) <= SOLVE_TOL


# test_solver.cpp known answers through the device Krylov engine (callable seam)

def _t(a):
    import torch

    return torch.from_numpy(np.asarray(a, np.complex128)).cuda()


def test_device_gmres_identity_one_iteration():
    from paper_2201_12050_b200 import gmres

    b = np.array([1 + 2j, -0.5, 3j])
    rep = gmres(lambda v: v, b, tol=1e-12)
    assert rep.converged and rep.iterations == 1
    assert np.linalg.norm(rep.solution - b) < 1e-12 * np.linalg.norm(b)


def test_device_gmres_diagonal():
    from paper_2201_12050_b200 import gmres

    dg = _t([2.0, 4.0])
    rep = gmres(lambda v: dg * v, np.array([2.0, 4.0], np.complex128), tol=1e-13)
    assert rep.converged
    np.testing.assert_allclose(rep.solution, [1, 1], atol=1e-12)


def test_device_gmres_random_dense_vs_direct_and_oracle():
    from paper_2201_12050_b200 import gmres

    rng = np.random.default_rng(11)
    n = 60
    a = np.eye(n) + 0.25 / np.sqrt(n) * crand(rng, n, n)
    b = crand(rng, n)
    at = _t(a)
    rep = gmres(lambda v: at @ v, b, tol=1e-12, restart=100, max_iter=300)
    assert rep.converged
    assert rel(rep.solution, np.linalg.solve(a, b)) < 1e-10
    x, its, conv, _ = O.gmres(lambda v: a @ v, b, tol=1e-12, restart=100, max_iter=300)
    assert abs(its - rep.iterations) <= 1


def test_device_gmres_restart_monotone_and_matches_oracle():
    from paper_2201_12050_b200 import gmres

    rng = np.random.default_rng(5)
    n, restart = 40, 7
    a = 2.0 * np.eye(n) + 0.3 / np.sqrt(n) * crand(rng, n, n)
    at = _t(a)
    b = np.ones(n, np.complex128)
    rep = gmres(lambda v: at @ v, b, tol=1e-11, restart=restart, max_iter=400)
    assert rep.converged and rep.iterations > restart
    h = rep.residual_history
    for i in range(1, len(h)):
        if i % restart:
            assert h[i] <= h[i - 1] * (1 + 1e-10)
    x, its, conv, _ = O.gmres(lambda v: a @ v, b, tol=1e-11, restart=restart, max_iter=400)
    assert abs(its - rep.iterations) <= 1 and rel(rep.solution, x) < SOLVE_TOL


def test_device_gmres_non_convergence_reported():
    from paper_2201_12050_b200 import gmres

    n = 30
    a = np.zeros((n, n))
    for i in range(n):
        a[(i + 1) % n, i] = 1.0
    at = _t(a)
    b = np.zeros(n, np.complex128)
    b[0] = 1
    rep = gmres(lambda v: at @ v, b, tol=1e-14, max_iter=5)
    assert not rep.converged and rep.iterations == 5


def test_device_gmres_nan_is_a_hard_error():
    from paper_2201_12050_b200 import gmres

    def bad(v):
        w = v.clone()
        w[2] = float("nan")
        return w

    with pytest.raises(RuntimeError, match="non-finite"):
        gmres(bad, np.ones(4, np.complex128))


def test_device_gmres_left_preconditioner():
    from paper_2201_12050_b200 import gmres

    n = 50
    d = 1.0 + 99.0 * np.arange(n) / (n - 1)
    dt = _t(d)
    b = np.ones(n, np.complex128)
    rep = gmres(lambda v: dt * v, b, tol=1e-12, preconditioner=lambda v: v / dt)
    assert rep.converged and rep.iterations == 1
    assert np.linalg.norm(d * rep.solution - b) / np.linalg.norm(b) < 1e-10


def test_fmm_gmres_zero_rhs_returns_immediately(ops, assembled):
    """src/solver.cpp:32-36: ||b|| == 0 -> converged, 0 iterations, x = 0, no history;
    also for one zero right-hand side inside a lockstep batch"""
    from paper_2201_12050_b200 import gmres

    sc, d = assembled(1, 0)
    rep = gmres(ops(d), np.zeros(d.N, np.complex128), tol=1e-6, restart=50, max_iter=100)
    assert rep.converged and rep.iterations == 0 and not np.any(rep.solution) and len(rep.residual_history) == 0
    b1 = sc.rhs(0)
    B = np.concatenate([b1, np.zeros(d.N, np.complex128), 2.0 * b1])
    reps = gmres(ops(d, max_rhs=3), B, tol=1e-8, restart=50, max_iter=200)
    assert reps[1].converged and reps[1].iterations == 0 and not np.any(reps[1].solution)
    single = gmres(ops(d), b1, tol=1e-8, restart=50, max_iter=200)
    assert reps[0].iterations == single.iterations and rel(reps[0].solution, single.solution) <= SOLVE_TOL
    assert reps[2].iterations == single.iterations and rel(reps[2].solution, 2.0 * single.solution) <= SOLVE_TOL


def test_fmm_gmres_nan_rhs_is_a_hard_error(ops, assembled):
    from paper_2201_12050_b200 import gmres

    sc, d = assembled(1, 0)
    b = sc.rhs(0)
    b[5] = np.nan
    with pytest.raises(RuntimeError, match="non-finite"):
        gmres(ops(d), b, tol=1e-6, restart=50, max_iter=50)


# ---- multi-GPU decomposition, exercised on one GPU -------------------------------

@pytest.mark.parametrize("nranks", [2, 3, 8])
def test_partial_products_of_an_offset_partition_sum_to_the_product(ops, assembled, nranks):
    """fpbem_cu_fmm_set_partition: every rank's partial product (own near-field
    offsets; rank 0 adds P2M/M2L/L2P) summed over ranks == the full product.
    Ranks run one after another on one GPU (no rank waits on another)."""
    sc, d = assembled(3, 2)
    rng = np.random.default_rng(3)
    p = uvec(rng, d.N)
    full = ops(d).matvec(p)
    total = np.zeros_like(full)
    for r in range(nranks):
        op = ops(d)
        op.set_partition(r, nranks)
        total += op.matvec(p)
        op.close()
    assert rel(total, full) < 1e-13
    assert rel(total, O.OracleFmm(d).matvec(p)) <= MATVEC_TOL


def test_nccl_communicator_single_rank_path(ops, assembled):
    """The NCCL all-reduce path of apply() with a 1-rank communicator."""
    import os

    import torch.distributed as dist

    from paper_2201_12050_b200.fmm import Communicator

    sc, d = assembled(2, 2)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29517")
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        comm = Communicator(device=0)
        op = ops(d)
        p = uvec(np.random.default_rng(9), d.N)
        y0 = op.matvec(p)
        op.set_comm(comm)
        assert np.array_equal(op.matvec(p), y0)
        from paper_2201_12050_b200 import gmres

        rep = gmres(op, sc.rhs(0), tol=1e-6, restart=50, max_iter=400)
        assert rep.converged
        op.set_comm(None)
        op.close()
        comm.close()
    finally:
        dist.destroy_process_group()


# ---- half space: folded image and the block-Hankel image pair (§8 a9) -----------

def _halfspace_scene(counts, pitch, lift, refl, n_t=4):
    from paper_2201_12050_b200 import Scene

    sc = Scene.custom("cube_sphere", [0.1, 2], counts, pitch, 2 * np.pi * 400 / 343)
    sc.shift_cell([0, 0, lift])
    sc.set_halfspace(2, 0.0, refl)
    return sc, sc.assemble_fmm(n_t)


@pytest.mark.parametrize("counts,pitch,lift", [((1, 2, 2), (0.0, 0.35, 0.35), 0.25),
                                               ((2, 1, 3), (0.35, 0.0, 0.35), 0.3),
                                               ((3, 2, 4), (0.35, 0.35, 0.35), 0.25)])
def test_hankel_image_pair_matches_oracle(ops, counts, pitch, lift):
    """FmmOperators::matvec with near_field_image + k_image_spectrum (src/fmm.cpp:262-269)."""
    sc, d = _halfspace_scene(counts, pitch, lift, 0.8 - 0.3j)
    assert d.mirrored_level == 2 and d.n_hat + d.n_far_hat > 0
    op = ops(d)
    rng = np.random.default_rng(sum(counts))
    p = uvec(rng, d.N)
    ora = O.OracleFmm(d)
    assert rel(op.matvec(p), ora.matvec(p)) <= MATVEC_TOL
    assert op.stored_bytes() == 16 * ((d.n_near + d.n_hat) * d.n_dof ** 2
                                      + 2 * int(np.prod(ora.sizes)) * 625 + 2 * 25 * d.n_dof)


def test_hankel_image_pair_near_dense_and_gmres(ops):
    """reference test_fmm.cpp:264-278 on the device: < 1e-5 vs dense at n_t = 8; GMRES parity."""
    from paper_2201_12050_b200 import gmres

    sc, d = _halfspace_scene((1, 2, 2), (0.0, 0.35, 0.35), 0.25, 1.0, n_t=8)
    op = ops(d)
    rng = np.random.default_rng(5)
    p = uvec(rng, d.N)
    assert rel(op.matvec(p), sc.dense() @ p) < 1e-5
    b = sc.rhs(0)
    rep = gmres(op, b, tol=1e-8, restart=50, max_iter=300)
    x, its, conv, _ = O.OracleFmm(d).gmres(b, tol=1e-8, restart=50, max_iter=300)
    assert rep.converged and conv and abs(rep.iterations - its) <= 1
    assert rel(rep.solution, x) <= SOLVE_TOL


def test_prebuilt_image_spectrum_is_accepted(ops):
    """the reference's k_image_spectrum handed over as lambda_hat"""
    sc, d = _halfspace_scene((1, 2, 2), (0.0, 0.35, 0.35), 0.25, 0.6)
    ora = O.OracleFmm(d)
    op = ops(d, lambda_=ora.lambda_, fft_sizes=ora.sizes, lambda_hat=ora.image_lambda)
    p = uvec(np.random.default_rng(11), d.N)
    assert rel(op.matvec(p), ora.matvec(p)) <= MATVEC_TOL


def test_folded_half_space_matches_oracle(ops):
    sc, d = _halfspace_scene((2, 2, 1), (0.35, 0.35, 0.0), 0.6, 0.9 + 0.2j)
    assert d.mirrored_level == -1
    p = uvec(np.random.default_rng(6), d.N)
    assert rel(ops(d).matvec(p), O.OracleFmm(d).matvec(p)) <= MATVEC_TOL


def test_balanced_partition_partials_sum_to_product(ops, assembled):
    """set_partition with a rank-0 deficit (the far field's measured cost in
    pair equivalents): partial products still sum to the product, rank 0 owns
    fewer pairs"""
    sc, d = assembled(2, 2)
    op = ops(d)
    far = op.far_pairs()
    assert far > 0.0
    p = uvec(np.random.default_rng(31), d.N)
    full = op.matvec(p)
    total = np.zeros_like(full)
    sizes = []
    for r in range(4):
        op.set_partition(r, 4, far_pairs=max(far, 3.0))
        lo, hi, f = op.partition()
        sizes.append(hi - lo)
        total += op.matvec(p)
    assert rel(total, full) < 1e-13
    assert sizes[0] < sizes[1]


def test_hankel_partition_sums_to_product(ops):
    sc, d = _halfspace_scene((3, 2, 4), (0.35, 0.35, 0.35), 0.25, 0.7)
    p = uvec(np.random.default_rng(8), d.N)
    full = ops(d).matvec(p)
    total = np.zeros_like(full)
    for r in range(3):
        op = ops(d)
        op.set_partition(r, 3)
        total += op.matvec(p)
    assert rel(total, full) < 1e-13


# ---- near-field assembly on the device ---------------------

@pytest.mark.parametrize("cid,var", [(1, 0), (2, 2), (3, 2), (4, 2), (6, 8)])
def test_device_assembly_matches_host_assembly(ops, assembled, cid, var):
    from paper_2201_12050_b200.fmm import assemble_near_gpu

    sc, d = assembled(cid, var)
    blocks = assemble_near_gpu(sc, d)
    host = np.asarray(d.near_blocks)
    dev = blocks.cpu().numpy()
    assert rel(dev, host) < 1e-12
    # the operator built from device-assembled blocks
    p = uvec(np.random.default_rng(cid), d.N)
    assert rel(ops(d, near_blocks=blocks).matvec(p), O.OracleFmm(d).matvec(p)) < 1e-12


def test_device_assembly_of_half_space_images():
    from paper_2201_12050_b200.fmm import assemble_hat_gpu, assemble_near_gpu

    sc, d = _halfspace_scene((2, 2, 1), (0.35, 0.35, 0.0), 0.6, 0.9 + 0.2j)
    dev = assemble_near_gpu(sc, d, halfspace=(2, 0.0, 0.9 + 0.2j)).cpu().numpy()
    assert rel(dev, np.asarray(d.near_blocks)) < 1e-12
    sc, d = _halfspace_scene((1, 2, 2), (0.0, 0.35, 0.35), 0.25, 0.8 - 0.3j)
    dev = assemble_hat_gpu(sc, d, (2, 0.0, 0.8 - 0.3j)).cpu().numpy()
    assert rel(dev, np.asarray(d.hat_blocks)) < 1e-12


# ---- M2L bank on the device ---------------------------------

@pytest.mark.parametrize("cid,var", [(1, 0), (2, 2), (3, 2), (4, 2), (5, 2)])
def test_device_m2l_bank_matches_host_bank(ops, assembled, cid, var):
    """fpbem_cu_m2l_bank = TranslationTable::m2l over the far offsets (host
    restatement, pinned by tests/test_host.py), and the operator built from the
    device bank reproduces the oracle product."""
    from paper_2201_12050_b200.fmm import assemble_far_gpu

    sc, d = assembled(cid, var)
    far, far_hat = assemble_far_gpu(sc, d)
    assert far_hat is None and far.shape == (d.n_far, d.n_coef, d.n_coef)
    if d.n_far:  # the shrunk variants can have every offset near
        assert rel(far.cpu().numpy(), np.asarray(d.far_blocks)) < 1e-13
    p = uvec(np.random.default_rng(cid + 40), d.N)
    assert rel(ops(d, far_blocks=far).matvec(p), O.OracleFmm(d).matvec(p)) <= MATVEC_TOL


def test_device_m2l_bank_without_host_bank_values(ops):
    """skip_near_values + skip_far_values: the host only classifies; S and the
    K bank come from the device; the product equals the fully host-assembled one."""
    from paper_2201_12050_b200 import Scene
    from paper_2201_12050_b200.fmm import assemble_far_gpu, assemble_near_gpu

    sc = Scene(5, 2)
    full = sc.assemble_fmm(4)
    shape = sc.assemble_fmm(4, skip_near_values=True, skip_far_values=True)
    assert not shape.has_far_values and shape.far_blocks.shape[0] == 0
    far, _ = assemble_far_gpu(sc, shape)
    near = assemble_near_gpu(sc, shape)
    p = uvec(np.random.default_rng(3), full.N)
    assert rel(ops(shape, near_blocks=near, far_blocks=far).matvec(p), O.OracleFmm(full).matvec(p)) <= MATVEC_TOL


def test_device_m2l_bank_half_space_images(ops):
    """folded image term K(center - mirror(base)) P (src/fmm.cpp:186-190) and the
    split-half-space K_hat bank (src/fmm.cpp:204-242) on the device."""
    from paper_2201_12050_b200.fmm import assemble_far_gpu

    hs = (2, 0.0, 0.9 + 0.2j)
    sc, d = _halfspace_scene((4, 4, 1), (0.35, 0.35, 0.0), 0.6, hs[2])
    far, far_hat = assemble_far_gpu(sc, d, halfspace=hs)
    assert d.mirrored_level == -1 and far_hat is None and d.n_far > 0
    assert rel(far.cpu().numpy(), np.asarray(d.far_blocks)) < 1e-13
    p = uvec(np.random.default_rng(13), d.N)
    assert rel(ops(d, far_blocks=far).matvec(p), O.OracleFmm(d).matvec(p)) <= MATVEC_TOL
    hs = (2, 0.0, 0.8 - 0.3j)
    sc, d = _halfspace_scene((3, 2, 4), (0.35, 0.35, 0.35), 0.25, hs[2])
    far, far_hat = assemble_far_gpu(sc, d, halfspace=hs)
    assert d.mirrored_level == 2 and d.n_far_hat > 0
    assert rel(far.cpu().numpy(), np.asarray(d.far_blocks)) < 1e-13
    assert rel(far_hat.cpu().numpy(), np.asarray(d.far_hat_blocks)) < 1e-13
    p = uvec(np.random.default_rng(12), d.N)
    op = ops(d, far_blocks=far, far_hat_blocks=far_hat)
    assert rel(op.matvec(p), O.OracleFmm(d).matvec(p)) <= MATVEC_TOL


def test_device_m2l_bank_other_orders():
    """n_t = 1..8 against the host TranslationTable (host.m2l_block)."""
    from paper_2201_12050_b200.fmm import m2l_bank_gpu
    from paper_2201_12050_b200.host import m2l_block

    rng = np.random.default_rng(21)
    deltas = rng.uniform(-3, 3, (7, 3)) + np.array([0.0, 0.0, 4.0])
    for n_t in (1, 2, 5, 8):
        dev = m2l_bank_gpu(n_t, 3.1, deltas).cpu().numpy()
        for s, dl in enumerate(deltas):
            host = m2l_block(n_t, dl, 3.1)
            assert rel(dev[s].T, host) < 1e-13


# ---- field evaluation on the device --------------------------

def _field_points(sc, n_far=12):
    """a grid in front of the array plus points within 3 element diameters of the
    surface (the adaptive-subdivision branch of the influence quadrature)"""
    from paper_2201_12050_b200.host import grid_points

    c = sc.cell()
    lo = np.min(c["centroid"], axis=0)
    hi = np.max(c["centroid"], axis=0) + np.asarray(sc.pitch) * (np.asarray(sc.counts) - 1)
    far = grid_points(lo - 0.6, hi + 0.6, (3, 2, 2))[:n_far]
    i = np.arange(0, len(c["centroid"]), max(1, len(c["centroid"]) // 5))[:5]
    near = c["centroid"][i] + 0.3 * c["diameter"][i, None] * c["normal"][i]  # just outside the surface
    return np.concatenate([far, near])


@pytest.mark.parametrize("cid,var", [(1, 0), (2, 2), (5, 2)])
def test_device_field_matches_host_evaluate_field(cid, var):
    from paper_2201_12050_b200 import Scene
    from paper_2201_12050_b200.fmm import evaluate_field_gpu

    sc = Scene(cid, var)
    pts = _field_points(sc)
    sol = uvec(np.random.default_rng(cid + 70), sc.N)
    host = sc.field_host(sol, pts)
    dev = evaluate_field_gpu(sc, sol, pts)
    assert rel(dev, host) < 1e-12
    # device pointers in, device tensor out
    import torch

    dev_t = evaluate_field_gpu(sc, torch.from_numpy(sol).cuda(), pts)
    assert dev_t.is_cuda and rel(dev_t.cpu().numpy(), host) < 1e-12


def test_device_field_with_half_space_images():
    from paper_2201_12050_b200.fmm import evaluate_field_gpu

    sc, d = _halfspace_scene((2, 2, 1), (0.35, 0.35, 0.0), 0.6, 0.9 + 0.2j)
    assert sc.halfspace is not None
    pts = _field_points(sc)
    sol = uvec(np.random.default_rng(77), sc.N)
    assert rel(evaluate_field_gpu(sc, sol, pts), sc.field_host(sol, pts)) < 1e-12


def test_solve_then_field_then_insertion_loss(ops, assembled):
    """run_scene's post-solve chain (src/scene.cpp:456-465) on the device:
    GMRES solution -> evaluate_field -> insertion_loss, against the host chain."""
    from paper_2201_12050_b200 import gmres
    from paper_2201_12050_b200.fmm import evaluate_field_gpu
    from paper_2201_12050_b200.host import insertion_loss

    sc, d = assembled(1, 0)
    rep = gmres(ops(d), sc.rhs(0), tol=1e-8, restart=50, max_iter=300)
    assert rep.converged
    pts = _field_points(sc)
    p_inc = sc.incident(pts)
    p_dev = evaluate_field_gpu(sc, rep.solution, pts, p_incident=p_inc)
    p_host = sc.field_host(rep.solution, pts)
    assert rel(p_dev, p_host) < 1e-12
    assert abs(insertion_loss(p_inc, p_dev) - insertion_loss(p_inc, p_host)) < 1e-10


# ---- lockstep batched GMRES (cfg5's 64 right-hand sides) -------------------------

def test_batched_gmres_matches_per_rhs_oracle_with_restarts(ops, assembled):
    """several RHS in lockstep, restart 7 so every RHS runs several cycles and the
    RHS leave the batch at different iterations; each equals its own single-RHS
    reference solve (src/solver.cpp:21-123)."""
    from paper_2201_12050_b200 import gmres

    sc, d = assembled(5, 2)
    dirs = [[1, 0, 0], [0, 0.6, 0.8], [0.3, -0.4, 0.866], [-1, 0.2, 0.1], [0, 0, 1]]
    sc.set_sources([1] * len(dirs), dirs)
    b = np.concatenate([sc.rhs(r) for r in range(len(dirs))])
    op = ops(d, max_rhs=len(dirs))
    reps = gmres(op, b, tol=1e-7, restart=7, max_iter=400)
    ora = O.OracleFmm(d)
    its = []
    for r in range(len(dirs)):
        x, it, conv, hist = ora.gmres(b[r * d.N:(r + 1) * d.N], tol=1e-7, restart=7, max_iter=400)
        assert reps[r].converged == conv
        assert abs(reps[r].iterations - it) <= 1
        assert rel(reps[r].solution, x) <= SOLVE_TOL
        its.append(it)
    assert len(set(its)) > 1  # the RHS really leave the batch at different times


def test_rhs_sharded_solve_single_process_equals_batch(ops, assembled):
    """gmres_sharded without a process group: one shard = the lockstep batch"""
    from paper_2201_12050_b200 import gmres
    from paper_2201_12050_b200.fmm import gmres_sharded

    sc, d = assembled(5, 2)
    dirs = [[1, 0, 0], [0, 0.6, 0.8], [0.3, -0.4, 0.866]]
    sc.set_sources([1] * len(dirs), dirs)
    B = np.concatenate([sc.rhs(r) for r in range(len(dirs))])
    op = ops(d, max_rhs=len(dirs))
    sharded = gmres_sharded(op, B, len(dirs), tol=1e-7, restart=30, max_iter=300)
    batch = gmres(op, B, tol=1e-7, restart=30, max_iter=300)
    for a, b in zip(sharded, batch):
        assert a.iterations == b.iterations and a.converged == b.converged
        assert np.array_equal(a.solution, b.solution)


def test_batched_gmres_equals_sequential_solves(ops, assembled):
    import os

    from paper_2201_12050_b200 import gmres

    sc, d = assembled(3, 2)
    sc.set_sources([1, 1, 1], [[1, 1, 1], [1, 0, 0], [0, 1, 0]])
    b = np.concatenate([sc.rhs(r) for r in range(3)])
    op = ops(d, max_rhs=3)
    batched = gmres(op, b, tol=1e-6, restart=20, max_iter=300)
    os.environ["FPBEM_GMRES_BATCHED"] = "0"
    try:
        seq = gmres(op, b, tol=1e-6, restart=20, max_iter=300)
    finally:
        del os.environ["FPBEM_GMRES_BATCHED"]
    for a, s in zip(batched, seq):
        assert abs(a.iterations - s.iterations) <= 1
        assert rel(a.solution, s.solution) < 1e-10


def test_batched_gmres_max_iter_and_nan(ops, assembled):
    from paper_2201_12050_b200 import gmres

    sc, d = assembled(1, 0)
    b = np.concatenate([sc.rhs(0), 2 * sc.rhs(0)])
    reps = gmres(ops(d, max_rhs=2), b, tol=1e-14, restart=5, max_iter=12)
    assert all(r.iterations == 12 and not r.converged for r in reps)
    b[d.N + 7] = np.nan
    with pytest.raises(RuntimeError, match="non-finite"):
        gmres(ops(d, max_rhs=2), b, tol=1e-6, restart=5, max_iter=12)


# ---- BASELINE sizes ----------------------------------------------------------------

@pytest.mark.parametrize("cid", [2, 3, 4])
def test_full_size_matvec_parity_and_properties(ops, cid):
    """configs[cid-1] at the stated size: operator assembled on the GPU, product
    against the oracle (seed = config id), linearity, determinism, and the
    8-way pair partition summing back to the product."""
    from paper_2201_12050_b200 import Scene
    from paper_2201_12050_b200.fmm import assemble_near_gpu

    sc = Scene(cid, 0)
    d = sc.assemble_fmm(4, skip_near_values=True)
    near = assemble_near_gpu(sc, d)

    class WithNear:
        def __init__(self, d, blocks):
            self._d, self.near_blocks = d, blocks

        def __getattr__(self, k):
            return getattr(self._d, k)

    full = WithNear(d, near.cpu().numpy())
    op = ops(d, near_blocks=near)
    rng = np.random.default_rng(cid)
    p, q = uvec(rng, d.N), uvec(rng, d.N)
    y = op.matvec(p)
    assert rel(y, O.OracleFmm(full).matvec(p)) <= MATVEC_TOL
    assert np.array_equal(y, op.matvec(p))
    a = 0.7 - 0.2j
    assert rel(op.matvec(a * p + q), a * y + op.matvec(q)) < 1e-13
    if cid == 3:
        total = np.zeros_like(y)
        for r in range(8):
            part = ops(d, near_blocks=near)
            part.set_partition(r, 8)
            total += part.matvec(p)
            part.close()
        assert rel(total, y) < 1e-13
