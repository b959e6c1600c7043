"""CPU tests of the z-slab decomposition's host logic (no GPU, no library):
slab geometry, per-rank RAS box sets, and the halo / allreduce hooks over a
real 2-process gloo group and over the thread emulation."""

import os
import socket
import threading

import numpy as np
import pytest
import torch

from paper_2007_04560_b200.exceptions import PartitionError
from paper_2007_04560_b200.grid import BoundaryCondition, Grid
from paper_2007_04560_b200.linalg import partition
from paper_2007_04560_b200.slab import ThreadGroup, TorchDistComm, split_grid


def test_split_grid_geometry():
    g = Grid((16, 12, 32), (1.0, 2.0, 4.0), BoundaryCondition.NEUMANN)
    slabs = [split_grid(g, 4, r) for r in range(4)]
    assert [s.z0 for s in slabs] == [0, 8, 16, 24]
    assert all(s.counts == (16, 12, 8) for s in slabs)
    assert all(abs(s.spacing[2] - g.spacing[2]) < 1e-15 for s in slabs)
    assert slabs[0].wall_lo and not slabs[0].wall_hi and slabs[3].wall_hi
    assert slabs[1].n_store == 16 * 12 * (8 + 4)
    assert slabs[2].global_grid() == g
    p = split_grid(Grid((8, 8, 16), (1.0, 1.0, 1.0), BoundaryCondition.PERIODIC), 2, 1)
    assert not p.wall_lo and not p.wall_hi
    with pytest.raises(PartitionError):
        split_grid(g, 5, 0)


@pytest.mark.parametrize("bc", [BoundaryCondition.PERIODIC, BoundaryCondition.NEUMANN])
def test_slab_partition_tiles_the_global_partition(bc):
    g = Grid((16, 16, 32), (1.0, 1.0, 1.0), bc)
    glob = partition(g, 64, 1)
    seen = []
    for r in range(4):
        s = split_grid(g, 4, r)
        d = partition(s, 64, 1)
        lo = d.owned_lo.copy()
        hi = d.owned_hi.copy()
        lo[:, 2] += s.z0
        hi[:, 2] += s.z0
        seen += [tuple(a) + tuple(b) for a, b in zip(lo, hi)]
    ref = [tuple(a) + tuple(b) for a, b in zip(glob.owned_lo, glob.owned_hi)]
    assert seen == ref          # same boxes, same (z slowest) order


def test_slab_partition_rejects_straddling_boxes():
    g = Grid((8, 8, 16), (1.0, 1.0, 1.0), BoundaryCondition.PERIODIC)
    assert partition(split_grid(g, 2, 1), 2, 1).n_subdomains == 1    # boxes of 8 planes, slabs of 8
    with pytest.raises(PartitionError):
        partition(split_grid(g, 4, 0), 2, 1)                          # slabs of 4 cut boxes of 8


def _expected_ghosts(vals, plane, nz, zg, depth, rank, nranks, periodic):
    """Ghost planes a rank must receive, from the global plane values."""
    lo = rank - 1 if rank > 0 else (nranks - 1 if periodic else None)
    hi = rank + 1 if rank < nranks - 1 else (0 if periodic else None)
    out = {}
    if lo is not None:
        out["bot"] = vals[lo][(zg + nz - depth) * plane:(zg + nz) * plane]
    if hi is not None:
        out["top"] = vals[hi][zg * plane:(zg + depth) * plane]
    return out


def _local_vector(rank, plane, nz, zg):
    v = torch.full(((nz + 2 * zg) * plane,), -1.0, dtype=torch.float64)
    for k in range(nz):
        v[(zg + k) * plane:(zg + k + 1) * plane] = 1000.0 * rank + k + torch.arange(plane) / plane
    return v


def _gloo_worker(rank, world, port, periodic, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = TorchDistComm(periodic)
        plane, nz, zg = 6, 4, 2
        res = {}
        for depth in (1, 2):
            v = _local_vector(rank, plane, nz, zg)
            comm.halo(v, plane, nz, zg, depth)
            res[depth] = v.numpy().copy()
        vals = np.array([rank + 1.0, -rank, 10.0 * rank])
        comm.allreduce(vals[:1], "sum")
        comm.allreduce(vals[1:2], "min")
        comm.allreduce(vals[2:], "max")
        q.put((rank, res, vals))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("periodic", [True, False])
def test_gloo_two_rank_halo_and_allreduce(periodic):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, periodic, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict()
    for _ in range(2):
        rank, res, vals = q.get(timeout=120)
        out[rank] = (res, vals)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    plane, nz, zg = 6, 4, 2
    base = [_local_vector(r, plane, nz, zg).numpy() for r in range(2)]
    for rank in range(2):
        res, vals = out[rank]
        assert vals[0] == 3.0 and vals[1] == -1.0 and vals[2] == 10.0
        for depth in (1, 2):
            exp = _expected_ghosts(base, plane, nz, zg, depth, rank, 2, periodic)
            got = res[depth]
            if "bot" in exp:
                np.testing.assert_array_equal(got[(zg - depth) * plane:zg * plane], exp["bot"])
            else:
                assert np.all(got[:zg * plane] == -1.0)
            if "top" in exp:
                np.testing.assert_array_equal(got[(zg + nz) * plane:(zg + nz + depth) * plane], exp["top"])
            else:
                assert np.all(got[(zg + nz) * plane:] == -1.0)
            # the interior is untouched
            np.testing.assert_array_equal(got[zg * plane:(zg + nz) * plane], base[rank][zg * plane:(zg + nz) * plane])


@pytest.mark.parametrize("nranks,periodic", [(3, True), (3, False), (1, True)])
def test_thread_comm_halo_and_allreduce(nranks, periodic):
    grp = ThreadGroup(nranks)
    plane, nz, zg = 5, 3, 2
    base = [_local_vector(r, plane, nz, zg).numpy() for r in range(nranks)]
    got = [None] * nranks
    sums = [None] * nranks

    def run(r):
        comm = grp.comm(r, periodic)
        v = torch.from_numpy(base[r].copy())
        comm.halo(v, plane, nz, zg, 2)
        got[r] = v.numpy()
        a = np.array([float(r), float(r)])
        comm.allreduce(a, "sum")
        sums[r] = a

    ts = [threading.Thread(target=run, args=(r,)) for r in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for r in range(nranks):
        exp = _expected_ghosts(base, plane, nz, zg, 2, r, nranks, periodic)
        if "bot" in exp:
            np.testing.assert_array_equal(got[r][:zg * plane], exp["bot"])
        if "top" in exp:
            np.testing.assert_array_equal(got[r][(zg + nz) * plane:], exp["top"])
        assert sums[r][0] == sum(range(nranks))


def _nccl_id_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2007_04560_b200.slab import NcclComm
        comm = NcclComm(periodic=True)
        ids = [comm.unique_id(), comm.unique_id()]
        q.put((rank, ids, comm.lower(), comm.upper(), comm.nccl_path))
    finally:
        dist.destroy_process_group()


def test_nccl_unique_id_is_shared_over_gloo():
    """The in-library NCCL data plane's bootstrap on 2 CPU processes: rank 0
    draws an ncclUniqueId (dlopen of libnccl, no GPU needed), the gloo group
    broadcasts it, both ranks hold identical bytes; a second communicator gets
    a fresh id; the neighbour ranks are the periodic wrap."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_nccl_id_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(2):
        rank, ids, lo, hi, path = q.get(timeout=120)
        out[rank] = (ids, lo, hi)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ids0, ids1 = out[0][0], out[1][0]
    assert len(ids0[0]) == 128 and ids0 == ids1 and ids0[0] != ids0[1]
    assert out[0][1:] == (1, 1) and out[1][1:] == (0, 0)
