"""GPU parity of the lattice-convolution near field: the
Toeplitz blocks of BlockToeplitzMatrix::matvec (src/assembly.cpp:62-84)
embedded in an (M + max|o|) lattice and applied per Fourier mode, against the
CPU oracle's direct Toeplitz product and the direct device path, on identical
seeded inputs (matvec relative L2 <= 1e-10, GMRES iterations within +-1 and
solutions within 1e-8)."""
import numpy as np
import pytest

import oracle as O
from conftest import rel
from test_gpu_parity import SMALL_SCENES, all_offsets, crand, toeplitz_only, uvec

pytestmark = pytest.mark.gpu

MATVEC_TOL = 1e-10
SOLVE_TOL = 1e-8


@pytest.fixture(scope="module")
def ops():
    from paper_2201_12050_b200 import FmmOperators

    return FmmOperators


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


@pytest.mark.parametrize("counts", [(2, 1, 1), (3, 3, 1), (5, 1, 2), (2, 3, 2), (1, 16, 1), (4, 4, 4)])
@pytest.mark.parametrize("n", [3, 70, 130, 300])
def test_lattice_near_field_matches_oracle_and_direct(ops, counts, n):
    rng = np.random.default_rng(n + 3 * counts[0] + 5 * counts[1] + 7 * counts[2])
    d = toeplitz_only(rng, counts, n)
    lat = ops(d, near_path="lattice")
    path, sizes, nbytes, per_block, mask, dev = lat.near_path()
    R = np.abs(d.near_offsets).max(axis=0)
    assert path == "lattice" and per_block == 1 and mask == 1 and dev == -1.0
    assert sizes == tuple(int(m + r) if m > 1 else 1 for m, r in zip(counts, R))
    assert nbytes == 16 * n * n * int(np.prod(sizes))
    p = uvec(rng, d.N)
    y = lat.matvec(p)
    assert rel(y, O.toeplitz_matvec(counts, d.near_offsets, d.near_blocks, p)) <= MATVEC_TOL
    direct = ops(d, near_path="direct")
    assert direct.near_path()[0] == "direct"
    assert rel(y, direct.matvec(p)) <= MATVEC_TOL
    assert np.array_equal(y, lat.matvec(p))  # fixed-order sums: bitwise repeatable


def test_lattice_near_field_offset_subset_and_asymmetric_reach(ops):
    """absent offsets are zero blocks; the embedding length follows the
    largest |o| per axis (here 2 along x, 1 along y, 0 along z: the z axis
    needs no padding, the operator is block diagonal in z)"""
    rng = np.random.default_rng(12)
    counts, n = (6, 5, 3), 40
    offs = [o for o in all_offsets(counts) if abs(o[0]) <= 2 and abs(o[1]) <= 1 and o[2] == 0 and o != (2, 1, 0)]
    d = toeplitz_only(rng, counts, n)
    d.near_offsets = np.asarray(offs, np.int32)
    d.near_blocks = crand(rng, len(offs), n, n)
    op = ops(d, near_path="lattice")
    assert op.near_path()[1] == (8, 6, 3)
    p = uvec(rng, d.N)
    assert rel(op.matvec(p), O.toeplitz_matvec(counts, offs, d.near_blocks, p)) <= MATVEC_TOL


@pytest.mark.parametrize("cid,var", SMALL_SCENES)
def test_lattice_fmm_matvec_matches_oracle(ops, assembled, cid, var):
    sc, d = assembled(cid, var)
    if int(np.prod(d.counts)) == 1:
        with pytest.raises(RuntimeError, match="lattice"):
            ops(d, near_path="lattice")
        return
    op = ops(d, near_path="lattice")
    p = uvec(np.random.default_rng(cid), d.N)
    assert rel(op.matvec(p), O.OracleFmm(d).matvec(p)) <= MATVEC_TOL


@pytest.mark.parametrize("nrhs,inv", [(1, True), (2, True), (3, True), (9, True), (16, True), (70, True),
                                       (3, False), (8, False), (9, False)])
def test_lattice_multi_rhs_gemv_and_dmma(ops, assembled, nrhs, inv):
    """few right-hand sides: streaming per-mode GEMV (right-hand sides x modes
    per block <= 8: the icosphere's 8 modes per block allow 1); more: the
    per-mode products as DMMA GEMM tiles (rhs-major spectrum, image-mode tiles
    gathered / scattered through P_g). Every rhs equals its own single-rhs
    product and the oracle."""
    sc, d = assembled(3, 2)
    rng = np.random.default_rng(40 + nrhs)
    P = [uvec(rng, d.N) for _ in range(nrhs)]
    op = ops(d, max_rhs=nrhs, near_path="lattice", use_symmetries=inv)
    assert (op.near_path()[3] > 1) == inv
    y = op.matvec(np.concatenate(P))
    single = ops(d, near_path="lattice", use_symmetries=inv)
    ora = O.OracleFmm(d)
    for r in sorted({0, nrhs // 2, nrhs - 1}):
        yr = y[r * d.N:(r + 1) * d.N]
        assert rel(yr, single.matvec(P[r])) <= 1e-13
        assert rel(yr, ora.matvec(P[r])) <= MATVEC_TOL


@pytest.mark.parametrize("nranks", [2, 3, 8])
def test_lattice_mode_partition_sums_to_product(ops, assembled, nranks):
    """the lattice path partitions Fourier modes: every rank's partial product
    (its modes, zero elsewhere, through the inverse DFT) sums to the product"""
    sc, d = assembled(2, 2)
    op = ops(d, near_path="lattice")
    p = uvec(np.random.default_rng(9), d.N)
    full = op.matvec(p)
    total = np.zeros_like(full)
    covered = 0
    for r in range(nranks):
        op.set_partition(r, nranks)
        lo, hi, _ = op.partition()
        covered += hi - lo
        total += op.matvec(p)
    path, sizes, nbytes, per_block, mask, _ = op.near_path()
    assert per_block == 2  # the cylinder triangulation's point reflection: (qx, qy) and (-qx, -qy)
    assert covered == nbytes // (16 * d.n_dof ** 2)  # stored blocks (one per orbit of modes)
    assert rel(total, full) < 1e-13


def test_lattice_balanced_partition(ops, assembled):
    sc, d = assembled(2, 2)
    op = ops(d, near_path="lattice")
    far = op.far_pairs()  # far field in mode equivalents
    assert far > 0.0
    p = uvec(np.random.default_rng(17), d.N)
    full = op.matvec(p)
    total = np.zeros_like(full)
    sizes = []
    for r in range(4):
        op.set_partition(r, 4, far_pairs=max(far, 2.0))
        lo, hi, _ = op.partition()
        sizes.append(hi - lo)
        total += op.matvec(p)
    assert rel(total, full) < 1e-13
    assert sizes[0] < sizes[1]


@pytest.mark.parametrize("cid,var", [(1, 0), (3, 2), (5, 2)])
def test_lattice_gmres_matches_oracle(ops, assembled, cid, var):
    from paper_2201_12050_b200 import gmres

    sc, d = assembled(cid, var)
    b = sc.rhs(0)
    rep = gmres(ops(d, near_path="lattice"), b, tol=1e-6, restart=50, max_iter=400)
    x, its, conv, _ = O.OracleFmm(d).gmres(b, tol=1e-6, restart=50, max_iter=400)
    assert rep.converged == conv
    assert abs(rep.iterations - its) <= 1
    assert rel(rep.solution, x) <= SOLVE_TOL


def test_lattice_batched_gmres_matches_per_rhs_oracle(ops, assembled):
    from paper_2201_12050_b200 import gmres

    sc, d = assembled(3, 2)
    dirs = [[1, 0, 0], [0, 1, 0], [0.6, 0, 0.8], [0, 0.6, 0.8]]
    sc.set_sources([1] * len(dirs), dirs)
    b = np.concatenate([sc.rhs(i) for i in range(len(dirs))])
    reps = gmres(ops(d, max_rhs=len(dirs), near_path="lattice"), b, tol=1e-6, restart=20, max_iter=400)
    ora = O.OracleFmm(d)
    for r, rep in enumerate(reps):
        x, its, conv, _ = ora.gmres(b[r * d.N:(r + 1) * d.N], tol=1e-6, restart=20, max_iter=400)
        assert abs(rep.iterations - its) <= 1
        assert rel(rep.solution, x) <= SOLVE_TOL


def test_lattice_is_rejected_with_a_half_space_image_pair(ops):
    from test_gpu_parity import _halfspace_scene

    sc, d = _halfspace_scene((3, 2, 4), (0.35, 0.35, 0.35), 0.25, 0.7)
    with pytest.raises(RuntimeError, match="lattice"):
        ops(d, near_path="lattice")
    assert ops(d).near_path()[0] == "direct"  # auto never picks it there


def test_cost_model_choices_at_baseline_shapes(ops):
    """without mode pairing (all-zero blocks never verify the inversion) auto
    picks the lattice path for cfg2 (125 offsets over 4 x 32 cells of 1024 DOF:
    287 modes stream 4.8 GB against 67 GFLOP of direct GEMM) and the direct GEMM
    for cfg3 (19 offsets: 17^3 modes would stream 8 GB)"""
    from paper_2201_12050_b200 import Scene
    from test_gpu_parity import Data

    for cid, want in ((2, "lattice"), (3, "direct")):
        sc = Scene(cid, 0)
        near, far, _, _ = sc.classify()
        n, b = sc.n_dof, 25
        z = np.zeros
        d = Data(sc.counts, n, b, near, z((len(near), n, n)), far, z((len(far), b, b)), z((b, n)), z((n, b)))
        assert ops(d).near_path()[0] == want


@pytest.mark.parametrize("cid,path", [(2, "direct"), (2, "lattice"), (3, "direct"), (3, "lattice")])
def test_full_size_both_paths(ops, cid, path):
    """configs[1] (131,072 DOF) and configs[2] (1,310,720 DOF) at their stated
    sizes through either near path (lattice: mode pairs through the verified
    cell inversion): parity with the oracle (seed = config id), linearity,
    determinism, and a 4-way partition summing back to the product"""
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

    op = ops(d, near_blocks=near, near_path=path)
    info = op.near_path()
    assert info[0] == path
    if path == "lattice":
        assert info[3] > 1 and 0.0 <= info[5] <= 1e-12
    rng = np.random.default_rng(cid)
    p, q = uvec(rng, d.N), uvec(rng, d.N)
    y = op.matvec(p)
    assert rel(y, O.OracleFmm(WithNear(d, near.cpu().numpy())).matvec(p)) <= MATVEC_TOL
    assert np.array_equal(y, op.matvec(p))
    a = 0.7 - 0.2j
    assert rel(op.matvec(a * p + q), a * y + op.matvec(q)) < 1e-13
    total = np.zeros_like(y)
    for r in range(4):
        op.set_partition(r, 4)
        total += op.matvec(p)
    assert rel(total, y) < 1e-13


GROUPS = {"x": [1], "xy": [1, 2], "xyz": [1, 2, 4], "half-turn z": [3], "inversion": [7]}


def _closure(gens):
    G = {0}
    while True:
        new = {a ^ b for a in G | set(gens) for b in G | set(gens)} | G | set(gens)
        if new == G:
            return sorted(G)
        G = new


def _symmetric_toeplitz(rng, counts, n, gens, perturb=0.0):
    """random Toeplitz with S_{A_g o} = P_g S_o P_g for the group generated by
    the axis-sign maps gens, P_g commuting fixed-point-free involutions"""
    G = _closure(gens)
    k = len(gens)
    assert n % (1 << k) == 0
    idx = rng.permutation(n).reshape(-1, 1 << k)  # each row: one orbit of elements, bit b of the column = generator b
    gen_perm = {}
    for b, g in enumerate(gens):
        p = np.empty(n, np.int64)
        for row in idx:
            for c in range(1 << k):
                p[row[c]] = row[c ^ (1 << b)]
        gen_perm[g] = p
    perms = {0: np.arange(n)}
    for g in G:  # P of a product: compose the generators' permutations
        if g in perms:
            continue
        for a in list(perms):
            for b in gens:
                if a ^ b == g:
                    perms[g] = perms[a][gen_perm[b]]
    flip = lambda g, o: tuple(-c if g >> d & 1 else c for d, c in enumerate(o))  # noqa: E731
    offs = all_offsets(counts)
    blocks = {}
    for o in offs:
        if o in blocks:
            continue
        stab = [g for g in G if flip(g, o) == o]
        m = crand(rng, n, n)
        m = sum(m[np.ix_(perms[h], perms[h])] for h in stab) / len(stab)
        for g in G:
            blocks[flip(g, o)] = m[np.ix_(perms[g], perms[g])]
    d = toeplitz_only(rng, counts, n)
    d.near_offsets = np.asarray(offs, np.int32)
    d.near_blocks = np.stack([blocks[o] for o in offs])
    if perturb:
        d.near_blocks[0, 0, 0] += perturb
    d.cell_symmetries = [(g, perms[g].astype(np.int32)) for g in G if g]
    return d, G


def _orbits(sizes, G):
    seen, count, largest = set(), 0, 1
    for qz in range(sizes[2]):
        for qy in range(sizes[1]):
            for qx in range(sizes[0]):
                if (qx, qy, qz) in seen:
                    continue
                orb = {tuple((sizes[d] - c) % sizes[d] if g >> d & 1 else c for d, c in enumerate((qx, qy, qz)))
                       for g in G}
                seen |= orb
                count += 1
                largest = max(largest, len(orb))
    return count, largest


@pytest.mark.parametrize("counts,n,group", [((3, 3, 1), 64, "xy"), ((4, 2, 3), 40, "xyz"), ((1, 7, 1), 130, "inversion"),
                                            ((2, 2, 2), 8, "xyz"), ((5, 4, 1), 32, "half-turn z"), ((3, 2, 2), 24, "x")])
def test_lattice_mode_orbits_through_cell_symmetries(ops, counts, n, group):
    """S_{A_g o} = P_g S_o P_g for a group of axis-sign maps: one stored block per
    orbit of Fourier modes, the images through P_g; parity with the oracle and
    with the path that stores every mode"""
    rng = np.random.default_rng(n + sum(counts))
    d, G = _symmetric_toeplitz(rng, counts, n, GROUPS[group])
    op = ops(d, near_path="lattice")
    path, sizes, nbytes, per_block, mask, dev = op.near_path()
    assert mask == sum(1 << g for g in G) and dev <= 1e-15
    count, largest = _orbits(sizes, G)
    assert nbytes == 16 * n * n * count
    assert per_block == {1: 1, 2: 2, 3: 4, 4: 4}.get(largest, 8)
    p = uvec(rng, d.N)
    y = op.matvec(p)
    assert rel(y, O.toeplitz_matvec(counts, d.near_offsets, d.near_blocks, p)) <= MATVEC_TOL
    assert rel(y, ops(d, near_path="lattice", use_symmetries=False).matvec(p)) <= MATVEC_TOL
    P = [uvec(rng, d.N) for _ in range(11)]  # the DMMA path with image tiles
    Y = ops(d, max_rhs=11, near_path="lattice").matvec(np.concatenate(P))
    assert rel(Y[10 * d.N:], O.toeplitz_matvec(counts, d.near_offsets, d.near_blocks, P[10])) <= MATVEC_TOL


def test_lattice_symmetry_that_does_not_hold_is_refused(ops):
    """a symmetry the blocks do not satisfy (one entry perturbed) is measured
    and rejected: every mode stored, still the oracle's product"""
    rng = np.random.default_rng(77)
    d, G = _symmetric_toeplitz(rng, (3, 2, 1), 24, [1, 2], perturb=1e-6)
    op = ops(d, near_path="lattice")
    path, sizes, nbytes, per_block, mask, dev = op.near_path()
    assert dev > 1e-9 and per_block < 4
    p = uvec(rng, d.N)
    assert rel(op.matvec(p), O.toeplitz_matvec((3, 2, 1), d.near_offsets, d.near_blocks, p)) <= MATVEC_TOL


@pytest.mark.parametrize("cid,var,want", [(3, 2, 0xFF), (2, 2, 0x81), (4, 2, 0x81), (1, 1, None)])
def test_scene_symmetries_verified_on_assembled_blocks(ops, assembled, cid, var, want):
    """the generated meshes carry symmetry-consistent quadrature nodes: the
    icosphere verifies all 7 axis-sign maps, the cylinder triangulation (split
    by height) and the split box the inversion (rounding-level
    deviation); the reference's cube-sphere keeps
    whatever holds. Every product equals the oracle's."""
    sc, d = assembled(cid, var)
    op = ops(d, near_path="lattice")
    path, sizes, nbytes, per_block, mask, dev = op.near_path()
    if want is not None:
        assert mask == want and 0.0 <= dev <= 1e-12
    p = uvec(np.random.default_rng(cid), d.N)
    assert rel(op.matvec(p), O.OracleFmm(d).matvec(p)) <= MATVEC_TOL


def test_lattice_mode_partition_with_many_right_hand_sides(ops, assembled):
    """the DMMA job list of the lattice path covers only the rank's stored
    blocks: partial products of 12 right-hand sides over 3 ranks sum to the
    product, each right-hand side equal to the oracle's"""
    sc, d = assembled(3, 2)
    rng = np.random.default_rng(123)
    P = np.concatenate([uvec(rng, d.N) for _ in range(12)])
    op = ops(d, max_rhs=12, near_path="lattice")
    full = op.matvec(P)
    total = np.zeros_like(full)
    for r in range(3):
        op.set_partition(r, 3)
        total += op.matvec(P)
    assert rel(total, full) < 1e-13
    ora = O.OracleFmm(d)
    for k in (0, 11):
        assert rel(full[k * d.N:(k + 1) * d.N], ora.matvec(P[k * d.N:(k + 1) * d.N])) <= MATVEC_TOL


@pytest.mark.parametrize("counts,n,group,nrhs", [((4, 2, 3), 40, "xyz", 1), ((3, 3, 2), 64, "xy", 2),
                                                 ((2, 3, 2), 320, "xyz", 1), ((3, 1, 2), 512, "x", 4)])
def test_tensor_core_mode_product_with_partition(ops, counts, n, group, nrhs):
    """the DMMA mode product with the bulk-copy block ring (n % 8 == 0, up to 8
    columns per stored block = right-hand sides x images): each right-hand
    side equals the oracle's product, and partial products of a 3-way
    stored-block partition sum to the full product"""
    rng = np.random.default_rng(n + nrhs)
    d, G = _symmetric_toeplitz(rng, counts, n, GROUPS[group])
    op = ops(d, near_path="lattice", max_rhs=nrhs)
    P = np.concatenate([uvec(rng, d.N) for _ in range(nrhs)])
    full = op.matvec(P)
    for r in range(nrhs):
        ref = O.toeplitz_matvec(counts, d.near_offsets, d.near_blocks, P[r * d.N:(r + 1) * d.N])
        assert rel(full[r * d.N:(r + 1) * d.N], ref) <= MATVEC_TOL
    assert np.array_equal(full, op.matvec(P))
    total = np.zeros_like(full)
    for r in range(3):
        op.set_partition(r, 3)
        total += op.matvec(P)
    assert rel(total, full) < 1e-13


@pytest.mark.parametrize("cid,var", [(3, 2), (5, 2)])
def test_pipelined_host_product_equals_device_product(ops, assembled, cid, var):
    """The host-pointer product with the copies overlapped (z-plane slabs in on
    one copy stream, out on another, the x / y DFT passes slab by slab) runs
    the same kernels as the device-pointer product: bitwise equal, and equal
    to the oracle (src/fmm.cpp:246-271)."""
    import torch

    sc, d = assembled(cid, var)
    op = ops(d, near_path="lattice")
    p = uvec(np.random.default_rng(cid + 40), d.N)
    y_host = op.matvec(p)
    y_dev = op.matvec(torch.from_numpy(p).cuda()).cpu().numpy()
    torch.cuda.synchronize()
    assert np.array_equal(y_host, y_dev)
    assert rel(y_host, O.OracleFmm(d).matvec(p)) <= MATVEC_TOL
    for _ in range(3):  # repeated calls reuse the staging buffers and events
        assert np.array_equal(op.matvec(p), y_host)


def test_programmatic_dependent_launch_gives_the_same_bits(tmp_path):
    """FPBEM_PDL (0 off — the default —, 2 the DFT passes launched as programmatic dependents, 1 the mode
    product as well; griddepcontrol.wait in front of their first dependent access; read once per process,
    hence the subprocesses): the product and a GMRES solve of the shrunk cfg3 lattice are bitwise those
    of the ordinary launches, product after product."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    code = (
        "import sys, numpy as np\n"
        "from paper_2201_12050_b200 import Scene, FmmOperators, gmres\n"
        "d = Scene(3, 2).assemble_fmm(4)\n"
        "op = FmmOperators(d, near_path='lattice')\n"
        "rng = np.random.default_rng(5)\n"
        "p = rng.uniform(-1, 1, d.N) + 1j * rng.uniform(-1, 1, d.N)\n"
        "ys = [op.matvec(p) for _ in range(6)]\n"
        "assert all(np.array_equal(ys[0], y) for y in ys)\n"
        "rep = gmres(op, p, tol=1e-8, restart=20, max_iter=200)\n"
        "np.save(sys.argv[1], np.concatenate([ys[0], np.asarray(rep.solution), [rep.iterations]]))\n"
    )
    root = Path(__file__).resolve().parents[1]
    outs = []
    for pdl in ("0", "1", "2"):
        f = tmp_path / f"pdl{pdl}.npy"
        env = dict(os.environ, FPBEM_PDL=pdl, PYTHONPATH=str(root))
        r = subprocess.run([sys.executable, "-c", code, str(f)], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(f))
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
