"""Multi-rank decomposition of the matvec, on the CPU with
gloo (world size 2): the library's partition rule splits the near-field
(offset, target) pairs into equal contiguous ranges, rank 0 adds the far
field, the all-reduced partial products equal the single-process product.
The same rule drives the device path (fpbem_cu_fmm_set_partition /
set_comm); tests/test_gpu_parity.py checks the device partial products on
one GPU."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, cid, var, result_path):
    import torch
    import torch.distributed as dist

    import oracle as O
    from paper_2201_12050_b200 import Scene
    from paper_2201_12050_b200.fmm import near_pairs, partition_pairs

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc = Scene(cid, var)
    d = sc.assemble_fmm(4)
    pairs = near_pairs(d.counts, d.near_offsets)
    lo, hi = partition_pairs(len(pairs), world, rank)
    rng = np.random.default_rng(cid)
    x = rng.uniform(-1, 1, d.N) + 1j * rng.uniform(-1, 1, d.N)
    n = d.n_dof
    X = x.reshape(-1, n)
    part = np.zeros_like(X)
    for s, t, src in pairs[lo:hi]:  # this rank's near-field pairs: y_t += S_s p_src
        part[t] += d.near_blocks[s].T @ X[src]
    part = part.reshape(-1)
    if rank == 0:  # rank 0 adds the far field (P2M, M2L, L2P)
        full = O.OracleFmm(d).matvec(x)
        part = part + (full - O.toeplitz_matvec(d.counts, d.near_offsets, d.near_blocks, x))
    t_ = torch.from_numpy(part.view(np.float64).copy())
    dist.all_reduce(t_)
    y = t_.numpy().view(np.complex128)
    if rank == 0:
        ref = O.OracleFmm(d).matvec(x)
        err = np.linalg.norm(y - ref) / np.linalg.norm(ref)
        sizes = [partition_pairs(len(pairs), world, r) for r in range(world)]
        np.save(result_path, np.array([err, hi - lo, min(h - l for l, h in sizes), max(h - l for l, h in sizes)]))
    dist.destroy_process_group()


@pytest.mark.parametrize("cid,var", [(2, 2), (3, 2), (5, 2)])
def test_two_rank_offset_partition_matches_single_process(tmp_path, cid, var):
    import torch.multiprocessing as mp

    out = str(tmp_path / "res.npy")
    mp.spawn(_worker, args=(2, _free_port(), cid, var, out), nprocs=2, join=True)
    err, n_mine, lo, hi = np.load(out)
    assert err < 1e-13
    assert n_mine >= 1
    assert hi - lo <= 1  # equal shares of the near-field pairs


def test_partition_rule_covers_every_pair_once():
    from paper_2201_12050_b200.fmm import partition_pairs

    for n_pairs, world in [(8012, 8), (70336, 8), (22, 4), (3, 8), (0, 2)]:
        ranges = [partition_pairs(n_pairs, world, r) for r in range(world)]
        assert ranges[0][0] == 0 and ranges[-1][1] == n_pairs
        for (l0, h0), (l1, h1) in zip(ranges, ranges[1:]):
            assert h0 == l1
        sizes = [h - l for l, h in ranges]
        assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("n_pairs,world,far", [(8012, 8, 246.4), (70336, 8, 800.0), (8012, 2, 246.0),
                                               (22, 4, 100.0), (1274, 8, 0.4), (5, 3, 2.0)])
def test_balanced_partition_gives_rank0_its_far_field_deficit(n_pairs, world, far):
    """rank 0 runs the far field: it takes round(far) fewer pairs (never fewer
    than 0), ranks 1.. share the rest equally, every pair owned once"""
    from paper_2201_12050_b200.fmm import partition_pairs

    ranges = [partition_pairs(n_pairs, world, r, far) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == n_pairs
    for (l0, h0), (l1, h1) in zip(ranges, ranges[1:]):
        assert h0 == l1
    sizes = [h - l for l, h in ranges]
    assert min(sizes) >= 0 and max(sizes[1:]) - min(sizes[1:]) <= 1
    d = round(far)
    if d and sizes[0] > 0:  # rank 0 short by the deficit, within rounding of the equal shares
        assert abs((sizes[1] - sizes[0]) - d) <= 2 + d // (world - 1)
    # equal split when the far field is free
    assert partition_pairs(n_pairs, world, 0, 0.0) == (0, n_pairs // world)


def test_near_pairs_order_matches_the_device_count():
    from paper_2201_12050_b200 import Scene
    from paper_2201_12050_b200.fmm import near_pairs

    sc = Scene(2, 0)
    near, _, _, _ = sc.classify()
    assert len(near_pairs(sc.counts, near)) == 8012


def _sharded_worker(rank, world, port, result_path):
    import torch.distributed as dist

    import oracle as O
    from paper_2201_12050_b200 import Scene
    from paper_2201_12050_b200.fmm import gmres_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc = Scene(1, 2)
    d = sc.assemble_fmm(3)
    ora = O.OracleFmm(d)
    dirs = [[1, 0, 0], [0, 1, 0], [0, 0, 1], [0.6, 0.8, 0], [0, 0.6, 0.8]]
    sc.set_sources([1] * len(dirs), dirs)
    B = np.concatenate([sc.rhs(r) for r in range(len(dirs))])

    def solve(rhs):  # the oracle stands in for the device batch on this CPU-only box
        from paper_2201_12050_b200.fmm import SolveReport

        reps = []
        for r in rhs:
            x, its, conv, hist = ora.gmres(r, tol=1e-8, restart=20, max_iter=200)
            reps.append(SolveReport(x, list(hist), its, conv))
        return reps

    reps = gmres_sharded(None, B, len(dirs), solve=solve)
    if rank == 0:
        errs = []
        for r, rep in enumerate(reps):
            x, its, conv, _ = ora.gmres(B.reshape(len(dirs), -1)[r], tol=1e-8, restart=20, max_iter=200)
            errs.append(float(np.linalg.norm(rep.solution - x)) + abs(rep.iterations - its) + (rep.converged != conv))
        np.save(result_path, np.array(errs))
    dist.destroy_process_group()


def test_rhs_sharded_solves_gather_in_order(tmp_path):
    """cfg5's multi-GPU mode: independent solves round-robin over the
    ranks, gathered back in right-hand-side order on every rank"""
    import torch.multiprocessing as mp

    out = str(tmp_path / "sharded.npy")
    mp.spawn(_sharded_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    errs = np.load(out)
    assert len(errs) == 5 and np.all(errs == 0.0)


def test_rhs_shard_rule():
    from paper_2201_12050_b200.fmm import rhs_shard

    for n, world in [(64, 8), (64, 3), (5, 8), (0, 2)]:
        parts = [rhs_shard(n, world, r) for r in range(world)]
        assert sorted(i for p in parts for i in p) == list(range(n))
        assert max(map(len, parts)) - min(map(len, parts)) <= 1


# ---- distributed GMRES (fpbem_cu_gmres_dist), restated on the CPU ----------------

def _dist_gmres_model(dist, rank, world, counts, n_dof, partial, b, tol, restart, max_iter):
    """The device algorithm of csrc/gmres_dist.cu in numpy: rows in slabs of
    ceil(cells / world) whole cells, all-gather -> partial product ->
    reduce-scatter per product, classical Gram-Schmidt passes with one
    all-reduce each and the reference's second-pass test, the reference's
    Givens / restart control flow (src/solver.cpp:21-123)."""
    import torch

    cells = int(np.prod(counts))
    N = cells * n_dof
    ns = -(-cells // world) * n_dof
    lo, hi = min(N, rank * ns), min(N, (rank + 1) * ns)

    def allreduce(a):
        t = torch.from_numpy(np.ascontiguousarray(a).view(np.float64).copy())
        dist.all_reduce(t)
        return t.numpy().view(np.complex128)

    def gather(v):
        full = np.zeros(world * ns, np.complex128)
        full[rank * ns:rank * ns + ns] = v
        return allreduce(full)

    def product(v):
        y = np.zeros(world * ns, np.complex128)
        y[:N] = partial(gather(v)[:N])
        return allreduce(y)[rank * ns:rank * ns + ns]

    bl = np.zeros(ns, np.complex128)
    bl[:hi - lo] = b[lo:hi]
    bnorm = np.sqrt(allreduce(np.array([np.vdot(bl, bl)]))[0].real)
    x = np.zeros(ns, np.complex128)
    its, hist = 0, []
    if bnorm == 0:
        return gather(x)[:N], 0, True, hist, (lo, hi)
    m = restart
    r, rnorm, conv = bl, bnorm, False
    while its < max_iter:
        V = [r / rnorm]
        H = np.zeros((m + 1, m), np.complex128)
        g = np.zeros(m + 1, np.complex128)
        g[0] = rnorm
        cs, sn = np.zeros(m), np.zeros(m, np.complex128)
        j = 0
        while j < m and its < max_iter:
            w = product(V[j])
            Vm = np.array(V)
            red = allreduce(np.concatenate([Vm.conj() @ w, [np.vdot(w, w)]]))
            h, pre2 = red[:-1], red[-1].real
            w = w - h @ Vm
            post2 = allreduce(np.array([np.vdot(w, w)]))[0].real
            if np.sqrt(post2) < 0.5 * np.sqrt(pre2):
                hc = allreduce(Vm.conj() @ w)
                w = w - hc @ Vm
                h = h + hc
                post2 = allreduce(np.array([np.vdot(w, w)]))[0].real
            hlast = np.sqrt(post2)
            H[:j + 1, j] = h
            H[j + 1, j] = hlast
            V.append(w / hlast if hlast > 0 else w)
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -np.conj(sn[i]) * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            a, bb = H[j, j], abs(H[j + 1, j])
            den = np.hypot(abs(a), bb)
            if den == 0:
                cs[j], sn[j] = 1.0, 0.0
            elif abs(a) == 0:
                cs[j], sn[j] = 0.0, 1.0
            else:
                cs[j], sn[j] = abs(a) / den, (a / abs(a)) * np.conj(H[j + 1, j]) / den
            H[j, j] = cs[j] * a + sn[j] * H[j + 1, j]
            H[j + 1, j] = 0
            g[j + 1] = -np.conj(sn[j]) * g[j]
            g[j] = cs[j] * g[j]
            its += 1
            est = abs(g[j + 1]) / bnorm
            hist.append(est)
            j += 1
            if est <= tol or hlast == 0:
                break
        y = np.zeros(j, np.complex128)
        for i in range(j - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:j] @ y[i + 1:j]) / H[i, i]
        x = x + y @ np.array(V[:j])
        r = bl - product(x)
        rnorm = np.sqrt(allreduce(np.array([np.vdot(r, r)]))[0].real)
        if rnorm / bnorm <= tol:
            conv = True
            break
    conv = conv or rnorm / bnorm <= tol
    return gather(x)[:N], its, conv, hist, (lo, hi)


def _dist_gmres_worker(rank, world, port, cid, var, restart, result_path):
    import torch.distributed as dist

    import oracle as O
    from paper_2201_12050_b200 import Scene
    from paper_2201_12050_b200.fmm import near_pairs, partition_pairs

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc = Scene(cid, var)
    d = sc.assemble_fmm(4)
    ora = O.OracleFmm(d)
    pairs = near_pairs(d.counts, d.near_offsets)
    lo, hi = partition_pairs(len(pairs), world, rank)
    n = d.n_dof

    def partial(x):  # this rank's near-field pairs; rank 0 adds the far field
        X = x.reshape(-1, n)
        part = np.zeros_like(X)
        for s, t, src in pairs[lo:hi]:
            part[t] += d.near_blocks[s].T @ X[src]
        part = part.reshape(-1)
        if rank == 0:
            part = part + (ora.matvec(x) - O.toeplitz_matvec(d.counts, d.near_offsets, d.near_blocks, x))
        return part

    b = sc.rhs(0)
    x, its, conv, hist, rows = _dist_gmres_model(dist, rank, world, d.counts, n, partial, b, 1e-6, restart, 400)
    if rank == 0:
        xo, its_o, conv_o, _ = ora.gmres(b, tol=1e-6, restart=restart, max_iter=400)
        np.save(result_path, np.array([float(np.linalg.norm(x - xo) / np.linalg.norm(xo)), its, its_o,
                                       float(conv), float(conv_o), rows[0], rows[1], d.N]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,cid,var,restart", [(2, 1, 0, 50), (3, 1, 1, 10), (3, 6, 8, 5)])
def test_distributed_gmres_restatement_matches_oracle(tmp_path, world, cid, var, restart):
    """The slab-distributed CGS GMRES of csrc/gmres_dist.cu, run in numpy over
    gloo ranks with the library's pair partition: iterations within +-1 and
    solution within 1e-8 of the oracle's MGS GMRES (BASELINE parity bar)."""
    import torch.multiprocessing as mp

    out = str(tmp_path / "dist.npy")
    mp.spawn(_dist_gmres_worker, args=(world, _free_port(), cid, var, restart, out), nprocs=world, join=True)
    err, its, its_o, conv, conv_o, lo, hi, N = np.load(out)
    assert conv == conv_o == 1.0
    assert abs(its - its_o) <= 1
    assert err <= 1e-8
    assert lo == 0 and 0 < hi <= N
