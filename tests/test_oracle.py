"""Pins the CPU oracle (oracle/fpbem_oracle.cpp) against the reference's own
known-answer tests for the hot path. The reference ships no stored vectors
(SURVEY.md §4, §8c); these are its hand-checked scalars, dense-expansion
oracles and solver known answers, re-run against the restatement:

  tests/test_structured.cpp:49-200  embedding, DFT, Toeplitz/Hankel products
  tests/test_solver.cpp:11-108       GMRES known answers
  acceptance_bench/bench.csv          operator byte counts (memory column)
"""
import numpy as np
import pytest

import oracle as O
from conftest import rel


def scalar_blocks(vals):
    return np.array([[[v]] for v in vals], np.complex128)


def all_offsets(counts):
    return [(x, y, z) for z in range(1 - counts[2], counts[2]) for y in range(1 - counts[1], counts[1])
            for x in range(1 - counts[0], counts[0])]


def random_toeplitz(rng, counts, b):
    offs = all_offsets(counts)
    blk = rng.standard_normal((len(offs), b, b)) + 1j * rng.standard_normal((len(offs), b, b))
    return offs, blk


def rvec(rng, n):
    return rng.standard_normal(n) + 1j * rng.standard_normal(n)


# --- test_structured.cpp -------------------------------------------------------

def test_embedding_order_of_one_level():
    # test_structured.cpp:49-68: offsets 0 -> 2, +1 -> 3, -1 -> 1 embed as column (2, 3, 1)
    sizes, lam = O.spectrum_build((2, 1, 1), [(0, 0, 0), (1, 0, 0), (-1, 0, 0)], scalar_blocks([2, 3, 1]))
    assert sizes == (3, 1, 1)
    column = O.dft3(lam, sizes, 1, +1) / 3.0
    np.testing.assert_allclose(column, [2, 3, 1], atol=1e-15)


def test_scalar_spectrum_by_hand():
    # test_structured.cpp:70-82: DFT of (2, 1, 1) is (4, 1, 1)
    _, lam = O.spectrum_build((2, 1, 1), [(0, 0, 0), (1, 0, 0), (-1, 0, 0)], scalar_blocks([2, 1, 1]))
    np.testing.assert_allclose(lam, [4, 1, 1], atol=1e-14)


def test_hand_checked_scalar_toeplitz_product():
    # test_structured.cpp:84-98: T = [[2,1],[3,2]], T (1,1) = (3, 5)
    offs, blk = [(0, 0, 0), (1, 0, 0), (-1, 0, 0)], scalar_blocks([2, 3, 1])
    sizes, lam = O.spectrum_build((2, 1, 1), offs, blk)
    p = np.array([1, 1], np.complex128)
    np.testing.assert_allclose(O.spectrum_matvec((2, 1, 1), sizes, 1, lam, p), [3, 5], atol=1e-14)
    np.testing.assert_allclose(O.toeplitz_matvec((2, 1, 1), offs, blk, p), [3, 5], atol=0)


def test_identity_unique_blocks_leave_vector_unchanged():
    # test_structured.cpp:100-111
    counts, b = (3, 2, 1), 4
    offs = all_offsets(counts)
    blk = np.zeros((len(offs), b, b), np.complex128)
    blk[offs.index((0, 0, 0))] = np.eye(b)
    p = rvec(np.random.default_rng(3), 3 * 2 * 4)
    sizes, lam = O.spectrum_build(counts, offs, blk)
    assert np.linalg.norm(O.spectrum_matvec(counts, sizes, b, lam, p) - p) < 1e-14 * np.linalg.norm(p)


def test_fft_product_equals_dense_expansion():
    # test_structured.cpp:113-120 (< 1e-13)
    rng = np.random.default_rng(17)
    counts, b = (3, 2, 1), 4
    offs, blk = random_toeplitz(rng, counts, b)
    dense = O.toeplitz_expand_dense(counts, offs, blk)
    p = rvec(rng, dense.shape[1])
    ref = dense @ p
    sizes, lam = O.spectrum_build(counts, offs, blk)
    assert rel(O.spectrum_matvec(counts, sizes, b, lam, p), ref) < 1e-13
    assert rel(O.toeplitz_matvec(counts, offs, blk, p), ref) < 1e-13


@pytest.mark.parametrize("mx", [1, 2, 3, 5])
@pytest.mark.parametrize("my", [1, 3])
@pytest.mark.parametrize("mz", [1, 2])
def test_all_level_count_combinations(mx, my, mz):
    # test_structured.cpp:122-140 (< 1e-12, linearity < 1e-13)
    rng = np.random.default_rng(100 + 10 * mx + 3 * my + mz)
    counts, b = (mx, my, mz), 3
    offs, blk = random_toeplitz(rng, counts, b)
    dense = O.toeplitz_expand_dense(counts, offs, blk)
    sizes, lam = O.spectrum_build(counts, offs, blk)
    p, q = rvec(rng, dense.shape[1]), rvec(rng, dense.shape[1])
    ref = dense @ p
    assert rel(O.spectrum_matvec(counts, sizes, b, lam, p), ref) < 1e-12
    a = 0.7 - 0.4j
    lhs = O.spectrum_matvec(counts, sizes, b, lam, a * p + q)
    rhs = a * O.spectrum_matvec(counts, sizes, b, lam, p) + O.spectrum_matvec(counts, sizes, b, lam, q)
    assert rel(lhs, rhs) < 1e-13


def hankel_via_spectrum(counts, level, indices, blk, p):
    """hankel_spectrum + hankel_matvec (src/structured.cpp:185-203)."""
    offs = np.array(indices).copy()
    offs[:, level] -= counts[level] - 1
    sizes, lam = O.spectrum_build(counts, offs, blk)
    return O.spectrum_matvec(counts, sizes, blk.shape[-1], lam, O.mirror_permute(counts, level, blk.shape[-1], p))


def test_hand_checked_scalar_hankel_product():
    # test_structured.cpp:142-161
    a, b_, c = 1.5, -0.5 + 2j, 0.25 - 1j
    counts, idx = (1, 1, 2), [(0, 0, 0), (0, 0, 1), (0, 0, 2)]
    blk = scalar_blocks([a, b_, c])
    p = np.array([1, 0], np.complex128)
    direct = O.hankel_matvec(counts, 2, idx, blk, p)
    np.testing.assert_allclose(direct, [a, b_], atol=1e-15)
    assert np.linalg.norm(hankel_via_spectrum(counts, 2, idx, blk, p) - direct) < 1e-14


def test_mirror_permutation_is_an_involution():
    # test_structured.cpp:163-168
    counts = (3, 4, 2)
    p = rvec(np.random.default_rng(77), 3 * 4 * 2 * 5)
    assert np.array_equal(O.mirror_permute(counts, 1, 5, O.mirror_permute(counts, 1, 5, p)), p)


def test_random_block_hankel_against_dense():
    # test_structured.cpp:170-190
    rng = np.random.default_rng(31)
    counts, b, level = (2, 3, 1), 3, 1
    idx = [(ox, s, 0) for s in range(5) for ox in (-1, 0, 1)]
    blk = rng.standard_normal((len(idx), b, b)) + 1j * rng.standard_normal((len(idx), b, b))
    n = 2 * 3 * b
    dense = np.zeros((n, n), np.complex128)
    cells = [(x, y, 0) for y in range(3) for x in range(2)]
    for ti, t in enumerate(cells):
        for si, s in enumerate(cells):
            key = (t[0] - s[0], t[1] + s[1], 0)
            if key in idx:
                dense[ti * b:(ti + 1) * b, si * b:(si + 1) * b] = blk[idx.index(key)].T
    p = rvec(rng, n)
    ref = dense @ p
    assert rel(O.hankel_matvec(counts, level, idx, blk, p), ref) < 1e-13
    assert rel(hankel_via_spectrum(counts, level, idx, blk, p), ref) < 1e-13


def test_padded_prime_embedding_length():
    # test_structured.cpp:192-200: 2M-1 = 31 is prime, padded to 32
    rng = np.random.default_rng(41)
    counts, b = (1, 16, 1), 2
    offs, blk = random_toeplitz(rng, counts, b)
    sizes, lam = O.spectrum_build(counts, offs, blk)
    assert sizes == (1, 32, 1)
    dense = O.toeplitz_expand_dense(counts, offs, blk)
    p = rvec(rng, dense.shape[1])
    assert rel(O.spectrum_matvec(counts, sizes, b, lam, p), dense @ p) < 1e-12


@pytest.mark.parametrize("length", [2, 3, 5, 7, 15, 16, 31, 32, 63, 64, 441 // 7, 512, 125])
def test_dft_matches_numpy(length):
    """The restated FFTW DFT against numpy's pocketfft (independent)."""
    rng = np.random.default_rng(length)
    x = rvec(rng, length * 3)
    got = O.dft3(x, (length, 1, 1), 3, -1).reshape(length, 3)
    ref = np.fft.fft(x.reshape(length, 3), axis=0)
    assert rel(got, ref) < 1e-14
    back = O.dft3(got.reshape(-1), (length, 1, 1), 3, +1).reshape(length, 3) / length
    assert rel(back, x.reshape(length, 3)) < 1e-14


def test_dft3_matches_numpy_fftn():
    rng = np.random.default_rng(9)
    sizes, h = (7, 9, 4), 5
    x = rvec(rng, int(np.prod(sizes)) * h)
    got = O.dft3(x, sizes, h, -1).reshape(sizes[2], sizes[1], sizes[0], h)
    ref = np.fft.fftn(x.reshape(sizes[2], sizes[1], sizes[0], h), axes=(0, 1, 2))
    assert rel(got, ref) < 1e-14


@pytest.mark.parametrize("lengths", [(15, 1, 1), (7, 63, 1), (8, 8, 8)])
def test_any_embedding_length_is_exact(lengths):
    """SURVEY finding 7: any L >= 2M-1 gives the same product (code pads 7-smooth, SPEC says 2M-1)."""
    rng = np.random.default_rng(5)
    counts = tuple((l + 1) // 2 if l > 1 else 1 for l in lengths)
    offs, blk = random_toeplitz(rng, counts, 2)
    dense = O.toeplitz_expand_dense(counts, offs, blk)
    p = rvec(rng, dense.shape[1])
    for sizes in (tuple(2 * m - 1 for m in counts), tuple(3 * m if m > 1 else 1 for m in counts)):
        s, lam = O.spectrum_build(counts, offs, blk, sizes)
        assert s == sizes
        assert rel(O.spectrum_matvec(counts, s, 2, lam, p), dense @ p) < 1e-12


# --- test_solver.cpp -----------------------------------------------------------

def test_gmres_identity_converges_in_one_iteration():
    b = np.array([1 + 2j, -0.5, 3j])
    x, its, conv, _ = O.gmres(lambda v: v, b, tol=1e-12)
    assert conv and its == 1
    assert np.linalg.norm(x - b) < 1e-12 * np.linalg.norm(b)


def test_gmres_diagonal_operator():
    b = np.array([2.0, 4.0], np.complex128)
    x, its, conv, _ = O.gmres(lambda v: v * np.array([2.0, 4.0]), b, tol=1e-13)
    assert conv
    np.testing.assert_allclose(x, [1, 1], atol=1e-12)


def test_gmres_random_dense_against_direct_solve():
    rng = np.random.default_rng(11)
    n = 60
    a = np.eye(n) + 0.25 / np.sqrt(n) * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    b = rvec(rng, n)
    x, its, conv, _ = O.gmres(lambda v: a @ v, b, tol=1e-12, restart=100, max_iter=300)
    direct = np.linalg.solve(a, b)
    assert conv
    assert rel(x, direct) < 1e-10
    assert np.linalg.norm(b - a @ x) / np.linalg.norm(b) <= 1e-12


def test_gmres_restart_history_monotone_per_cycle():
    rng = np.random.default_rng(5)
    n, restart = 40, 7
    a = 2.0 * np.eye(n) + 0.3 / np.sqrt(n) * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    b = np.ones(n, np.complex128)
    x, its, conv, hist = O.gmres(lambda v: a @ v, b, tol=1e-11, restart=restart, max_iter=400)
    assert conv and its > restart
    for i in range(1, len(hist)):
        if i % restart == 0:
            continue
        assert hist[i] <= hist[i - 1] * (1 + 1e-10)


def test_gmres_non_convergence_is_reported():
    n = 30
    a = np.zeros((n, n))
    for i in range(n):
        a[(i + 1) % n, i] = 1.0
    b = np.zeros(n, np.complex128)
    b[0] = 1.0
    x, its, conv, _ = O.gmres(lambda v: a @ v, b, tol=1e-14, max_iter=5)
    assert not conv and its == 5


def test_gmres_nan_is_a_hard_error():
    def bad(v):
        w = v.copy()
        w[2] = np.nan
        return w

    with pytest.raises(RuntimeError, match="non-finite"):
        O.gmres(bad, np.ones(4, np.complex128))


def test_gmres_left_preconditioner():
    n = 50
    d = 1.0 + 99.0 * np.arange(n) / (n - 1)
    b = np.ones(n, np.complex128)
    x, its, conv, _ = O.gmres(lambda v: d * v, b, tol=1e-12, preconditioner=lambda v: v / d)
    assert conv and its == 1
    assert np.linalg.norm(d * x - b) / np.linalg.norm(b) < 1e-10


def test_gmres_zero_rhs():
    x, its, conv, hist = O.gmres(lambda v: 2 * v, np.zeros(5, np.complex128))
    assert conv and its == 0 and not hist and not np.any(x)


# --- acceptance_bench/bench.csv ---------------------------------------------------

@pytest.mark.parametrize("my,fmpbem_bytes,pbem_bytes", [(8, 196848, 138240), (16, 366848, 294912),
                                                        (32, 676848, 580608), (64, 1326848, 1179648)])
def test_bench_csv_operator_bytes(my, fmpbem_bytes, pbem_bytes):
    """bench.csv memory column: stored_bytes of the fmpbem operators (3 near
    blocks of the 24-element cell + spectrum + U0 + V0) and of the pbem
    spectrum, reproduced exactly from the offset classification and the
    7-smooth embedding length."""
    from paper_2201_12050_b200.host import Scene

    sc = Scene(6, my)  # criterion-6 scene: cube-sphere r=0.1 ref 2 on 1 x My x 1, pitch 0.35
    near, far, _, _ = sc.classify()
    n = sc.n_dof
    assert n == 24
    q = O.fft_friendly(2 * my - 1)
    assert len(near) * n * n * 16 + q * 25 * 25 * 16 + 2 * 25 * n * 16 == fmpbem_bytes
    assert q * n * n * 16 == pbem_bytes
