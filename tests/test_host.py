"""Host operator producer (libfpbem_host.so): the reference's assembly-side
known answers (tests/test_fmm.cpp, tests/test_assembly.cpp,
tests/test_specfun.cpp, tests/acceptance.cpp criterion 2), checked on the
CPU with the oracle as the matvec. Independent references: scipy's spherical
Bessel functions, dense assembly, finite differences."""
import numpy as np
import pytest

import oracle as O
from conftest import rel
from paper_2201_12050_b200 import host as H
from paper_2201_12050_b200.host import Scene


def test_spherical_bessel_against_scipy():
    sp = pytest.importorskip("scipy.special")
    for x in [1e-3, 0.3, 1.0, 4.5, 12.0, 40.0]:
        j, y = H.sph_bessel(12, x)
        for n in range(13):
            assert abs(j[n] - sp.spherical_jn(n, x)) <= 1e-13 * max(1.0, abs(sp.spherical_jn(n, x)))
            if x > 0.2 or n < 6:
                assert abs(y[n] - sp.spherical_yn(n, x)) <= 1e-12 * abs(sp.spherical_yn(n, x))


def test_wigner3j_known_values():
    assert H.wigner3j(1, 1, 0, 0, 0, 0) == pytest.approx(-1 / np.sqrt(3), abs=1e-15)
    assert H.wigner3j(1, 1, 2, 0, 0, 0) == pytest.approx(np.sqrt(2 / 15), abs=1e-15)
    assert H.wigner3j(2, 2, 2, 0, 0, 0) == pytest.approx(-np.sqrt(2 / 35), abs=1e-15)
    assert H.wigner3j(1, 1, 1, 0, 0, 0) == 0.0  # odd J selection rule
    assert H.wigner3j(2, 1, 1, 1, 0, 0) == 0.0  # m sum


def test_solid_harmonic_gradients_by_finite_differences():
    k, v = 3.7, np.array([0.21, -0.13, 0.34])
    val, dx, dy, dz = H.solid_regular_gradients(4, v, k)
    h = 1e-6
    for axis, d in enumerate((dx, dy, dz)):
        e = np.zeros(3)
        e[axis] = h
        fd = (H.solid_regular_gradients(4, v + e, k)[0] - H.solid_regular_gradients(4, v - e, k)[0]) / (2 * h)
        assert np.max(np.abs(fd - d)) < 1e-7


def test_m2l_block_degree_zero_is_the_singular_harmonic():
    # tests/test_fmm.cpp:110-114: n_t = 0 block equals O_0^0(delta; k)
    k = 2 * np.pi * 500 / 343
    b = H.m2l_block(0, [0.5, 0, 0], k)
    o = H.solid_singular(0, [0.5, 0, 0], k)
    assert abs(b[0, 0] - o[0]) < 1e-14
    # j0 + i y0 = -i e^{ikr}/(kr)
    kr = k * 0.5
    assert abs(o[0] - (-1j) * np.exp(1j * kr) / kr) < 1e-14


def test_generators_match_the_configs():
    counts = {1: (320, (8, 1, 1)), 2: (1024, (4, 32, 1)), 3: (320, (16, 16, 16)), 4: (3680, (1, 256, 1)),
              5: (320, (32, 32, 4))}
    for cid, (n, c) in counts.items():
        sc = Scene(cid, 0)
        assert sc.n_dof == n and sc.counts == c
    cell = Scene(2, 0).cell()
    assert np.all(cell["area"] > 0) and np.all(cell["nv"] == 3)
    # closed surfaces: sum of area-weighted outward normals vanishes
    for cid in (1, 2, 3, 4):
        c = Scene(cid, 0).cell()
        assert np.linalg.norm((c["normal"] * c["area"][:, None]).sum(0)) < 1e-12
    assert Scene(5, 0).n_rhs == 64


def test_offset_classification_matches_survey_appendix_a():
    expect = {1: (3, 12), 2: (125, 316), 3: (19, 29772), 4: (5, 506), 5: (19, 27764)}
    for cid, (nn, nf) in expect.items():
        near, far, _, _ = Scene(cid, 0).classify()
        assert (len(near), len(far)) == (nn, nf)


def test_near_and_far_supports_are_complementary():
    # tests/test_fmm.cpp:191-204: cube-sphere r=0.1 refinement 1, pitch 0.35
    for counts in [(5, 5, 1), (3, 1, 2), (2, 2, 2)]:
        sc = Scene.custom("cube_sphere", [0.1, 1], counts, [0.35] * 3, 1.0)
        near, far, _, _ = sc.classify()
        total = np.prod([2 * c - 1 for c in counts])
        assert len(near) + len(far) == total
        if counts == (5, 5, 1):
            assert (len(near), len(far)) == (9, 72)
        # loop order z, y, x ascending (src/fmm.cpp:156-158)
        keys = [(o[2], o[1], o[0]) for o in near]
        assert keys == sorted(keys)


def test_single_cell_lattice_equals_dense():
    # tests/test_fmm.cpp:176-189: everything in the near field, == dense to 1e-14
    k = 2 * np.pi * 500 / 343
    sc = Scene.custom("cube_sphere", [0.1, 2], (1, 1, 1), [0.35] * 3, k)
    d = sc.assemble_fmm(4)
    assert d.n_near == 1 and d.n_far == 0
    rng = np.random.default_rng(0)
    p = rng.uniform(-1, 1, d.N) + 1j * rng.uniform(-1, 1, d.N)
    assert rel(O.OracleFmm(d).matvec(p), sc.dense() @ p) < 1e-14


def test_toeplitz_blocks_reconstruct_the_dense_system():
    # tests/test_assembly.cpp:85-101 on a 2x2 array
    k = 2 * np.pi * 500 / 343
    counts = (2, 2, 1)
    sc = Scene.custom("cube_sphere", [0.1, 2], counts, [0.35] * 3, k)
    offs = [(x, y, 0) for y in (-1, 0, 1) for x in (-1, 0, 1)]
    blocks = np.stack([sc.interaction_block(np.array(o) * 0.35, o == (0, 0, 0)).T for o in offs])
    rebuilt = O.toeplitz_expand_dense(counts, offs, blocks)
    dense = sc.dense()
    assert rel(rebuilt, dense) < 1e-13


def test_fmm_converges_to_dense_on_a_line_array():
    # tests/test_fmm.cpp:206-232: n_t 4 -> 8 decreases the error, < 1e-5 at 8
    k = 2 * np.pi * 500 / 343
    sc = Scene.custom("cube_sphere", [0.1, 2], (1, 3, 1), [0.35] * 3, k)
    dense = sc.dense()
    rng = np.random.default_rng(1)
    p = rng.uniform(-1, 1, sc.N) + 1j * rng.uniform(-1, 1, sc.N)
    ref = dense @ p
    errs = [rel(O.OracleFmm(sc.assemble_fmm(nt)).matvec(p), ref) for nt in (4, 8)]
    assert errs[1] < errs[0] and errs[1] < 1e-5


@pytest.mark.slow
def test_acceptance_criterion_2_fmpbem_accuracy():
    # tests/acceptance.cpp:108-127: 5x5 spheres, 96 elements, n_t = 4, 500 Hz, < 1e-4
    k = 2 * np.pi * 500 / 343
    sc = Scene.custom("cube_sphere", [0.1, 4], (5, 5, 1), [0.35] * 3, k)
    rng = np.random.default_rng(2)
    p = rng.standard_normal(sc.N) + 1j * rng.standard_normal(sc.N)
    err = rel(O.OracleFmm(sc.assemble_fmm(4)).matvec(p), sc.dense() @ p)
    assert err < 1e-4


def test_rhs_plane_wave_at_centroids():
    sc = Scene(1, 2)
    r = sc.rhs(0)
    c = sc.cell()
    k = sc.wavenumber
    # first cell: p = e^{ik x}, dp/dn_bie = ik d.(-n) e^{ikx}; alpha = -i/k
    x = c["centroid"][:, 0]
    ref = np.exp(1j * k * x) * (1 + (-1j / k) * 1j * k * (-c["normal"][:, 0]))
    assert rel(r[: sc.n_dof], ref) < 1e-14


# --- half space (tests/test_fmm.cpp:234-278) ---------------------------------------

def _raised_scene(counts, pitch, lift):
    k = 2 * np.pi * 400 / 343
    sc = Scene.custom("cube_sphere", [0.1, 2], counts, pitch, k)
    sc.shift_cell([0, 0, lift])
    return sc


def test_half_space_parallel_to_the_periodicity_folds_into_toeplitz():
    # test_fmm.cpp:234-262: mirror z=0 under a 2x2 array at z = 0.6, n_t = 8, < 1e-5 vs dense
    sc = _raised_scene((2, 2, 1), [0.35, 0.35, 0.0], 0.6)
    sc.set_halfspace(2, 0.0, 0.9 + 0.2j)
    d = sc.assemble_fmm(8)
    assert d.mirrored_level == -1 and d.n_hat == 0
    rng = np.random.default_rng(4)
    p = rng.uniform(-1, 1, sc.N) + 1j * rng.uniform(-1, 1, sc.N)
    assert rel(O.OracleFmm(d).matvec(p), sc.dense() @ p) < 1e-5
    # zero reflection gives the plain operators
    sc.set_halfspace(2, 0.0, 0.0)
    plain = O.OracleFmm(sc.assemble_fmm(4)).matvec(p)
    assert np.array_equal(plain, O.OracleFmm(sc.assemble_fmm(4)).matvec(p))


def test_half_space_perpendicular_to_the_periodicity_splits_into_hankel():
    # test_fmm.cpp:264-278: 1x2x2 array, mirror z=0 with the z axis periodic, n_t = 8, < 1e-5
    sc = _raised_scene((1, 2, 2), [0.0, 0.35, 0.35], 0.25)
    sc.set_halfspace(2, 0.0, 1.0)
    d = sc.assemble_fmm(8)
    assert d.mirrored_level == 2 and d.n_hat + d.n_far_hat == 3 * 3 * 1
    rng = np.random.default_rng(5)
    p = rng.uniform(-1, 1, sc.N) + 1j * rng.uniform(-1, 1, sc.N)
    assert rel(O.OracleFmm(d).matvec(p), sc.dense() @ p) < 1e-5


def test_mirrored_mesh_keeps_orientation_and_index():
    sc = Scene.custom("icosphere", [0.1, 1], (1, 1, 1), [0, 0, 0], 1.0)
    sc.shift_cell([0, 0, 0.5])
    c = sc.cell()
    # a mirrored triangle mesh through the dense image terms: a zero-reflection half space changes nothing
    sc.set_halfspace(2, 0.0, 0.0)
    a0 = sc.dense()
    sc.set_halfspace(2, 0.0, 1e-300)
    assert rel(sc.dense(), a0) < 1e-12
    assert c["nv"][0] == 3


@pytest.mark.parametrize("cid,var,want", [(3, 2, [1, 2, 3, 4, 5, 6, 7]), (2, 2, [7]), (4, 2, [7]),
                                          (1, 0, [1, 2, 3, 4, 5, 6, 7])])
def test_cell_symmetries_and_symmetric_quadrature_order(cid, var, want):
    """Scene.cell_symmetries (host C++ cell_symmetries): the axis-sign maps that
    map the generated unit cell onto itself, each with an element permutation;
    symmetrize_group gives every image element the images of its source's
    corners, reordered (b', a', c'[, d']) for orientation-reversing maps — the
    property that makes S_{A_g o}[P_g i, P_g j] = S_o[i, j] hold to rounding
    (DESIGN.md §3.1c)."""
    from paper_2201_12050_b200 import Scene

    sc = Scene(cid, var)
    syms = sc.cell_symmetries()
    assert [g for g, _ in syms] == want
    cell = sc.cell()
    cor, nv = cell["corners"], cell["nv"]
    pts = cor.reshape(-1, 3)
    ctr = 0.5 * (pts.min(axis=0) + pts.max(axis=0))
    tol = 1e-9 * np.linalg.norm(pts.max(axis=0) - pts.min(axis=0))
    for g, perm in syms:
        assert sorted(perm) == list(range(sc.n_dof))
        sign = np.array([-1.0 if g >> d & 1 else 1.0 for d in range(3)])
        img = ctr + sign * (cor - ctr)  # corners mapped by g, in the source's order
        reversing = bin(g).count("1") % 2 == 1
        for j in range(sc.n_dof):
            k = perm[j]
            if reversing:  # (b', a', c') / (b', a', d', c')
                order = [1, 0, 2, 2] if nv[j] == 3 else [1, 0, 3, 2]
                want_c = img[j][order]
            else:
                want_c = img[j]
            got = cor[k]
            ok = np.abs(got - want_c).max() < tol
            if not ok and not reversing and nv[j] == 4:  # a half-turn may map a quad to its own half-turn
                ok = np.abs(got - want_c[[2, 3, 0, 1]]).max() < tol
            assert ok, (g, j, k)


def test_reference_quad_cells_report_a_group_of_permutations():
    """the reference's own generators (wall cell, cube-sphere) are not reordered;
    their point-set symmetries still come back as a group of permutations (the
    device decides per map whether the blocks honour it)"""
    from paper_2201_12050_b200 import Scene

    for sc in (Scene.custom("wall", [1.0, 2.0, 0.1, 3], [1, 4, 1], [0.0, 1.0, 0.0], 2.0), Scene(1, 1)):
        syms = dict(sc.cell_symmetries())
        for g, perm in syms.items():
            assert sorted(perm) == list(range(sc.n_dof))
            assert np.array_equal(perm[perm], np.arange(sc.n_dof))  # axis-sign maps are involutions
            for h in syms:
                if h != g:
                    assert (g ^ h) in syms  # closed under composition
