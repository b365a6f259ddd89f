"""Multi-rank decomposition of the matvec, on the CPU with
gloo (world size 2): the library's offset partition rule splits the near
field, rank 0 adds the far field, the all-reduced partial products equal the
single-process product. The same rule drives the device path
(fpbem_cu_fmm_set_partition / set_comm); tests/test_gpu_parity.py checks the
device partial products on one GPU."""
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


class _Sub:
    """FmmData-like view with a subset of the near offsets."""

    def __init__(self, d, keep):
        self.counts, self.n_dof, self.n_coef = d.counts, d.n_dof, d.n_coef
        self.near_offsets = d.near_offsets[keep]
        self.near_blocks = d.near_blocks[keep]
        self.far_offsets, self.far_blocks, self.u0, self.v0 = d.far_offsets, d.far_blocks, d.u0, d.v0


def _pairs(d):
    m = d.counts
    return np.array([(m[0] - abs(o[0])) * (m[1] - abs(o[1])) * (m[2] - abs(o[2])) for o in d.near_offsets])


def _worker(rank, world, port, cid, var, result_path):
    import torch
    import torch.distributed as dist

    import oracle as O
    from paper_2201_12050_b200 import Scene
    from paper_2201_12050_b200.fmm import partition_offsets

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc = Scene(cid, var)
    d = sc.assemble_fmm(4)
    owner = partition_offsets(_pairs(d), world)
    mine = np.nonzero(owner == rank)[0]
    rng = np.random.default_rng(cid)
    x = rng.uniform(-1, 1, d.N) + 1j * rng.uniform(-1, 1, d.N)
    if rank == 0:
        part = O.OracleFmm(_Sub(d, mine)).matvec(x)  # own near offsets + far field
    else:
        part = O.toeplitz_matvec(d.counts, d.near_offsets[mine], d.near_blocks[mine], x)
    t = torch.from_numpy(part.view(np.float64).copy())
    dist.all_reduce(t)
    y = t.numpy().view(np.complex128)
    if rank == 0:
        ref = O.OracleFmm(d).matvec(x)
        err = np.linalg.norm(y - ref) / np.linalg.norm(ref)
        loads = [int(_pairs(d)[owner == r].sum()) for r in range(world)]
        np.save(result_path, np.array([err, len(mine), min(loads), max(loads)]))
    dist.destroy_process_group()


@pytest.mark.parametrize("cid,var", [(2, 2), (3, 2), (5, 2)])
def test_two_rank_offset_partition_matches_single_process(tmp_path, cid, var):
    import torch.multiprocessing as mp

    out = str(tmp_path / "res.npy")
    mp.spawn(_worker, args=(2, _free_port(), cid, var, out), nprocs=2, join=True)
    err, n_mine, lo, hi = np.load(out)
    assert err < 1e-13
    assert n_mine >= 1
    assert hi <= 1.5 * lo + 64  # work-balanced split of the near field


def test_partition_rule_is_balanced_and_deterministic():
    from paper_2201_12050_b200.fmm import partition_offsets

    work = np.array([128, 124, 120, 93, 93, 64, 48, 32, 31, 24, 24, 24])
    a = partition_offsets(work, 4)
    b = partition_offsets(work, 4)
    assert np.array_equal(a, b)
    loads = [work[a == r].sum() for r in range(4)]
    assert max(loads) - min(loads) <= work.max()
    assert set(a.tolist()) == {0, 1, 2, 3}
    assert np.array_equal(partition_offsets(work, 1), np.zeros(len(work), np.int32))
