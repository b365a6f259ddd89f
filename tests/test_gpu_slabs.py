"""Slab-distributed product (north_star "Fourier modes and
near-field cell slabs are split per GPU, and the FFT transpose is an NCCL
all-to-all"): every rank owns whole planes of cells along the slab axis and
applies FmmOperators::matvec (src/fmm.cpp:246-271) to its rows, with the
pruned lattice DFTs below the slab axis on its planes, one all-to-all per
direction, and the DFTs along the slab axis, the near-field block products and
the M2L on its columns. Ranks run as processes on one GPU exchanging through
the host-staged communicator (gloo all-reduce); the NCCL send/recv path runs
with a one-rank communicator. Parity: the slabs' products concatenated equal
the oracle's product (<= 1e-10) and the single-GPU product; the slab GMRES
(classical Gram-Schmidt with the reference's reorthogonalisation test) matches
the oracle's solver::gmres (iterations +-1, solution <= 1e-8)."""
import os
import pickle
import socket

import numpy as np
import pytest

import oracle as O
from conftest import rel
from test_gpu_parity import uvec

pytestmark = pytest.mark.gpu

MATVEC_TOL = 1e-10
SOLVE_TOL = 1e-8


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, cid, var, out_path):
    import torch.distributed as dist

    from paper_2201_12050_b200 import FmmOperators, Scene
    from paper_2201_12050_b200.fmm import HostCommunicator, gmres_distributed

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sc = Scene(cid, var)
        d = sc.assemble_fmm(4)
        op = FmmOperators(d, device=0, near_path="lattice")
        comm = HostCommunicator(0)
        op.set_slabs(comm)
        lo, hi = op.slab_rows()
        p = uvec(np.random.default_rng(cid), d.N)
        y = op.matvec_slab(p[lo:hi])
        rep = gmres_distributed(op, sc.rhs(0), tol=1e-6, restart=30, max_iter=600)
        res = (rank, (lo, hi), y, rep.iterations, rep.converged, rep.solution)
        gathered = [None] * world
        dist.all_gather_object(gathered, res)
        if rank == 0:
            with open(out_path, "wb") as f:
                pickle.dump(gathered, f)
        comm.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,cid,var", [(2, 3, 2), (3, 3, 2), (4, 3, 2), (2, 2, 2), (3, 5, 2), (3, 1, 2)])
def test_slab_product_and_solve_over_ranks(tmp_path, world, cid, var):
    """3-D lattices (z slabs: 4 x 4 x 4 spheres, 6 x 6 x 2), a 2-D lattice
    (y slabs: 4 x 8 cylinders) and a row (x slabs); 3 ranks on 4 planes leaves
    one rank a single plane, 3 ranks on 2 planes one rank none"""
    import torch.multiprocessing as mp

    from paper_2201_12050_b200 import FmmOperators, Scene

    out = str(tmp_path / "slabs.pkl")
    mp.spawn(_worker, args=(world, _free_port(), cid, var, out), nprocs=world, join=True)
    with open(out, "rb") as f:
        res = pickle.load(f)
    sc = Scene(cid, var)
    d = sc.assemble_fmm(4)
    p = uvec(np.random.default_rng(cid), d.N)
    rows = [r[1] for r in res]
    assert rows[0][0] == 0 and rows[-1][1] == d.N
    assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))  # slabs tile the rows in rank order
    y = np.concatenate([r[2] for r in res])
    ora = O.OracleFmm(d)
    assert rel(y, ora.matvec(p)) <= MATVEC_TOL
    assert rel(y, FmmOperators(d, near_path="lattice").matvec(p)) <= 1e-12
    x, its, conv, _ = ora.gmres(sc.rhs(0), tol=1e-6, restart=30, max_iter=600)
    for _, _, _, r_its, r_conv, sol in res:
        assert r_conv == conv and abs(r_its - its) <= 1
        assert rel(sol, x) <= SOLVE_TOL
        assert r_its == res[0][3] and np.array_equal(sol, res[0][5])  # identical on every rank


def test_slab_product_through_a_one_rank_nccl_communicator():
    """the grouped ncclSend / ncclRecv exchange with one rank: the slab is the
    whole vector, equal to the single-GPU product; device pointers too"""
    torch = pytest.importorskip("torch")
    import torch.distributed as dist

    from paper_2201_12050_b200 import FmmOperators, Scene
    from paper_2201_12050_b200.fmm import Communicator

    sc = Scene(3, 2)
    d = sc.assemble_fmm(4)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        op = FmmOperators(d, near_path="lattice")
        full = FmmOperators(d, near_path="lattice")
        comm = Communicator(device=0)
        op.set_slabs(comm)
        assert op.slab_rows() == (0, d.N)
        p = uvec(np.random.default_rng(3), d.N)
        y = op.matvec_slab(p)
        assert rel(y, full.matvec(p)) <= 1e-12
        yd = op.matvec_slab(torch.from_numpy(p).cuda())
        assert np.array_equal(yd.cpu().numpy(), y)
        comm.close()
    finally:
        dist.destroy_process_group()


def test_slab_plan_refuses_the_direct_path():
    from paper_2201_12050_b200 import FmmOperators, Scene

    d = Scene(4, 2).assemble_fmm(4)
    op = FmmOperators(d, near_path="direct")
    with pytest.raises(RuntimeError, match="lattice"):
        op.set_slabs(None)
    with pytest.raises(RuntimeError, match="slab plan"):
        op.slab_rows()


def test_slab_graph_replay_equals_eager_product():
    """the slab product replayed as CUDA graphs (the default with no or an NCCL
    communicator) equals the eager launch sequence bitwise (stage timing runs
    the eager path), for host and device pointers, repeatedly"""
    torch = pytest.importorskip("torch")
    from paper_2201_12050_b200 import FmmOperators, Scene

    sc = Scene(3, 2)
    d = sc.assemble_fmm(4)
    op = FmmOperators(d, near_path="lattice")
    op.set_slabs(None)
    p = uvec(np.random.default_rng(5), d.N)
    y_graph = op.matvec_slab(p)
    op.enable_stage_timing(True)
    y_eager = op.matvec_slab(p)
    op.enable_stage_timing(False)
    assert np.array_equal(y_graph, y_eager)
    xd = torch.from_numpy(p).cuda()
    for _ in range(3):
        assert np.array_equal(op.matvec_slab(xd).cpu().numpy(), y_graph)
    assert rel(y_graph, O.OracleFmm(d).matvec(p)) <= MATVEC_TOL


@pytest.mark.parametrize("P", [2, 3])
def test_simulated_communicator_counts_the_exchange(P):
    """fpbem_cu_comm_simulated: rank r of P alone on one GPU. Its two exchanges
    per product send exactly the bytes of the slab plan — forward: its planes
    of the other ranks' columns; backward: the other ranks' planes of its
    columns; both lattices (n values per near-field column entry, b per
    far-field one) — and its partial product stays finite. 3 ranks on the
    4 planes of a 4 x 4 x 4 lattice leave one rank without planes."""
    from paper_2201_12050_b200 import FmmOperators, Scene
    from paper_2201_12050_b200.fmm import SimulatedCommunicator

    sc = Scene(3, 2)
    d = sc.assemble_fmm(4)
    op = FmmOperators(d, near_path="lattice")
    Ln = op.near_path()[1]
    Lf = op.far_info()[0]
    n, b, Mz = d.n_dof, d.n_coef, d.counts[2]
    Cn, Cf = Ln[0] * Ln[1], Lf[0] * Lf[1]
    for r in range(P):
        comm = SimulatedCommunicator(0, P, r)
        op.set_slabs(comm)
        info = op.slab_info()
        assert info["rank"] == r and info["ranks"] == P and info["axis"] == 2
        lo, hi = op.slab_rows()
        assert hi - lo == info["planes"] * d.counts[0] * d.counts[1] * n
        comm.traffic(reset=True)
        y = op.matvec_slab(uvec(np.random.default_rng(r), d.N)[lo:hi])
        assert np.isfinite(y).all()
        sent, exchanges = comm.traffic(reset=True)
        assert exchanges == 2  # one grouped exchange per direction
        cn, cf, pl = info["near_modes"] // Ln[2], info["far_modes"] // Lf[2], info["planes"]
        fwd = pl * ((Cn - cn) * n + (Cf - cf) * b)
        bwd = (Mz - pl) * (cn * n + cf * b)
        assert sent == 16 * (fwd + bwd)
        op.set_slabs(None)
        comm.close()
