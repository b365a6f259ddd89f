"""Distributed GMRES (fpbem_cu_gmres_dist): Krylov basis split
over the ranks in slabs of whole cells, classical Gram-Schmidt passes with the
reference's reorthogonalisation test. Parity bar of BASELINE.json against the
oracle's MGS GMRES (src/solver.cpp:21-123): iterations within +-1, solutions
within 1e-8 relative.

Several ranks run as processes on ONE GPU through the host-staged
communicator over gloo (HostCommunicator): the collectives are host calls, no
kernel waits on another rank's kernel, so the ranks may time-share the GPU."""
import os
import pickle
import socket

import numpy as np
import pytest

import oracle as O
from conftest import rel

pytestmark = pytest.mark.gpu

SOLVE_TOL = 1e-8


def uvec(rng, n):
    return rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)


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


@pytest.mark.parametrize("cid,var,restart", [(1, 0, 50), (2, 2, 10), (3, 2, 50), (4, 2, 50), (5, 2, 50),
                                             (6, 8, 50)])
def test_dist_gmres_one_rank_matches_oracle(assembled, cid, var, restart):
    from paper_2201_12050_b200 import FmmOperators, gmres
    from paper_2201_12050_b200.fmm import dist_rows, gmres_distributed

    sc, d = assembled(cid, var)
    b = sc.rhs(0)
    op = FmmOperators(d)
    rep = gmres_distributed(op, b, tol=1e-6, restart=restart, max_iter=2000)
    x, its, conv, hist = O.OracleFmm(d).gmres(b, tol=1e-6, restart=restart, max_iter=2000)
    assert rep.converged == conv
    assert abs(rep.iterations - its) <= 1
    assert rel(rep.solution, x) <= SOLVE_TOL
    assert len(rep.residual_history) == rep.iterations
    n = min(len(hist), rep.iterations)
    assert rel(np.array(rep.residual_history[:n]), np.array(hist[:n])) < 1e-6
    assert dist_rows(op) == (0, d.N)
    mgs = gmres(op, b, tol=1e-6, restart=restart, max_iter=2000)  # the MGS device solver
    assert abs(mgs.iterations - rep.iterations) <= 1 and rel(mgs.solution, rep.solution) <= SOLVE_TOL


def test_dist_gmres_device_pointers_and_edge_cases(assembled):
    torch = pytest.importorskip("torch")
    from paper_2201_12050_b200 import FmmOperators
    from paper_2201_12050_b200.fmm import gmres_distributed

    sc, d = assembled(1, 0)
    op = FmmOperators(d)
    b = sc.rhs(0)
    host = gmres_distributed(op, b, tol=1e-6, restart=50, max_iter=400)
    dev = gmres_distributed(op, torch.from_numpy(b).cuda(), tol=1e-6, restart=50, max_iter=400)
    assert dev.iterations == host.iterations
    assert np.array_equal(dev.solution.cpu().numpy(), host.solution)  # fixed-order reductions
    # zero right-hand side: converged after 0 iterations, x = 0 (src/solver.cpp:32-36)
    z = gmres_distributed(op, np.zeros(d.N, np.complex128), tol=1e-6, restart=50, max_iter=400)
    assert z.converged and z.iterations == 0 and not np.any(z.solution) and not z.residual_history
    # max_iter caps the iterations, non-convergence is reported, not raised
    cap = gmres_distributed(op, b, tol=1e-14, restart=50, max_iter=3)
    assert cap.iterations == 3 and not cap.converged
    # a non-finite product is a hard error
    bad = b.copy()
    bad[7] = np.nan
    with pytest.raises(RuntimeError, match="non-finite"):
        gmres_distributed(op, bad, tol=1e-6, restart=50, max_iter=50)
    with pytest.raises(ValueError):
        gmres_distributed(op, np.zeros(d.N + 1, np.complex128))
    # a pair partition without a communicator would solve a partial operator
    op.set_partition(0, 2)
    with pytest.raises(RuntimeError, match="communicator"):
        gmres_distributed(op, b)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_worker(rank, world, port, cid, var, restart, out_path):
    import torch.distributed as dist

    from paper_2201_12050_b200 import FmmOperators, Scene
    from paper_2201_12050_b200.fmm import HostCommunicator, dist_rows, gmres_distributed

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sc = Scene(cid, var)
        d = sc.assemble_fmm(4)
        op = FmmOperators(d, device=0)
        comm = HostCommunicator(0)
        op.set_comm(comm)  # near-field pairs split, far field on rank 0
        p = uvec(np.random.default_rng(cid), d.N)
        y = op.matvec(p)  # partial products summed through the host all-reduce
        rep = gmres_distributed(op, sc.rhs(0), tol=1e-6, restart=restart, max_iter=2000)
        res = (rank, dist_rows(op), op.partition(), y, rep.iterations, rep.converged, rep.solution,
               rep.residual_history)
        gathered = [None] * world
        dist.all_gather_object(gathered, res)
        if rank == 0:
            with open(out_path, "wb") as f:
                pickle.dump(gathered, f)
        op.set_comm(None)
        comm.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,cid,var,restart", [(2, 3, 2, 50), (3, 2, 2, 10), (2, 5, 2, 50)])
def test_dist_gmres_over_ranks_matches_oracle(tmp_path, assembled, world, cid, var, restart):
    """world processes on one GPU: slabs cover the rows once, every rank
    returns the same full solution, the solve and the all-reduced product
    match the oracle."""
    import torch.multiprocessing as mp

    out = str(tmp_path / "dist.pkl")
    mp.spawn(_rank_worker, args=(world, _free_port(), cid, var, restart, out), nprocs=world, join=True)
    with open(out, "rb") as f:
        res = pickle.load(f)
    sc, d = assembled(cid, var)
    ora = O.OracleFmm(d)
    p = uvec(np.random.default_rng(cid), d.N)
    y_ref = ora.matvec(p)
    x, its, conv, _ = ora.gmres(sc.rhs(0), tol=1e-6, restart=restart, max_iter=2000)
    rows = [r[1] for r in res]
    assert rows[0][0] == 0 and rows[-1][1] == d.N
    assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
    assert all((hi - lo) % d.n_dof == 0 for lo, hi in rows)  # whole cells
    pairs = [r[2][:2] for r in res]
    assert all(a[1] == b[0] for a, b in zip(pairs, pairs[1:]))  # pair ranges tile the near field
    for rank, _, _, y, r_its, r_conv, sol, hist in res:
        assert rel(y, y_ref) <= 1e-10
        assert r_conv == conv and abs(r_its - its) <= 1
        assert rel(sol, x) <= SOLVE_TOL
        assert r_its == res[0][4] and np.array_equal(sol, res[0][6])  # identical on every rank


def test_dist_gmres_through_a_one_rank_nccl_communicator(assembled):
    """The NCCL collectives of the distributed solve (all-gather, reduce-scatter,
    all-reduce) with a communicator of one rank: same solve as no communicator."""
    import torch.distributed as dist

    from paper_2201_12050_b200 import FmmOperators
    from paper_2201_12050_b200.fmm import Communicator, gmres_distributed

    sc, d = assembled(3, 2)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        op = FmmOperators(d)
        alone = gmres_distributed(op, sc.rhs(0), tol=1e-6, restart=50, max_iter=400)
        comm = Communicator(device=0)
        op.set_comm(comm)
        rep = gmres_distributed(op, sc.rhs(0), tol=1e-6, restart=50, max_iter=400)
        assert rep.iterations == alone.iterations and np.array_equal(rep.solution, alone.solution)
        op.set_comm(None)
        comm.close()
    finally:
        dist.destroy_process_group()
