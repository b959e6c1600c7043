"""z-slab decomposition of a 3D grid across ranks (one GPU each).

SURVEY.md §8e: the grid is cut into equal slabs of whole z-planes; every rank
owns the RAS boxes inside its slab (box heights must divide the slab), keeps
two ghost planes below and above its interior (the residual and J·w are
radius-2 stencils by composition), and combines every reduction across ranks.
The library calls two host hooks (include/acch_b200.h, acch_set_comm): a halo
exchange of ghost planes and an allreduce of partial sums / minima.

Communicators:
* ``NcclComm`` -- the production data plane: the library itself runs NCCL
  send / recv of ghost planes and all-reduces on its stream (csrc/comm.cu),
  one process per GPU; the GMRES Arnoldi loop stays device-resident;
* ``TorchDistComm`` -- host hooks through torch.distributed point-to-point +
  all_reduce (NCCL over NVLink on GPUs, gloo on CPU tensors);
* ``ThreadComm`` -- ranks emulated as threads of one process (each with its
  own context and stream on one GPU), for validating the decomposition
  without several GPUs.  Ranks only meet in host-side barriers; no kernel
  ever waits for another rank's kernel.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np
import torch

from .exceptions import PartitionError
from .grid import Grid

GHOST = 2


@dataclass(frozen=True)
class SlabGrid(Grid):
    """This rank's slab: ``counts`` are the local (nx, ny, nz_local) with the
    global spacing; ``z0`` is the first global plane; ``nz_global`` the
    global plane count; ``ghost`` planes are stored on both sides."""

    nranks: int = 1
    rank: int = 0
    z0: int = 0
    nz_global: int = 0
    ghost: int = GHOST

    @property
    def wall_lo(self) -> bool:
        return (not self.periodic) and self.rank == 0

    @property
    def wall_hi(self) -> bool:
        return (not self.periodic) and self.rank == self.nranks - 1

    @property
    def plane_cells(self) -> int:
        return self.counts[0] * self.counts[1]

    @property
    def zoff(self) -> int:
        return self.ghost * self.plane_cells

    @property
    def n_store(self) -> int:
        return self.n_cells + 2 * self.zoff

    def global_grid(self) -> Grid:
        return Grid((self.counts[0], self.counts[1], self.nz_global),
                    (self.lengths[0], self.lengths[1], self.lengths[2] * self.nz_global / self.counts[2]), self.bc)

    def interior(self, t: torch.Tensor) -> torch.Tensor:
        """Interior part of a stored per-cell tensor (first dim = cells)."""
        return t[self.zoff:self.zoff + self.n_cells]


def split_grid(grid: Grid, nranks: int, rank: int, ghost: int = GHOST) -> SlabGrid:
    if grid.dim != 3:
        raise PartitionError("slab decomposition needs a 3D grid")
    nz = grid.counts[2]
    if nranks < 1 or nz % nranks:
        raise PartitionError(f"{nz} z-planes do not split evenly over {nranks} ranks")
    nzl = nz // nranks
    if nzl < max(2, ghost):
        raise PartitionError("slabs must be at least 2 planes deep")
    return SlabGrid((grid.counts[0], grid.counts[1], nzl),
                    (grid.lengths[0], grid.lengths[1], grid.lengths[2] * nzl / nz), grid.bc,
                    nranks=nranks, rank=rank, z0=rank * nzl, nz_global=nz, ghost=ghost)


def local_fields(slab: SlabGrid, u_global: np.ndarray, v_global: np.ndarray):
    """This rank's interior planes of global (nz, ny, nx) fields."""
    z0, z1 = slab.z0, slab.z0 + slab.counts[2]
    return u_global[z0:z1], v_global[z0:z1]


# ---------------------------------------------------------------------------
# communicators
# ---------------------------------------------------------------------------

_OPS = {0: "sum", 1: "min", 2: "max"}


class _DevBuf:
    """Zero-copy view of library-owned device memory (CUDA array interface)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3,
                                         "strides": None}


def _ghost_views(vec: torch.Tensor, plane: int, nz: int, zg: int, depth: int):
    """(bottom ghosts, top ghosts, bottom interior, top interior) views, each `depth` planes."""
    bot_g = vec[(zg - depth) * plane:zg * plane]
    top_g = vec[(zg + nz) * plane:(zg + nz + depth) * plane]
    bot_i = vec[zg * plane:(zg + depth) * plane]
    top_i = vec[(zg + nz - depth) * plane:(zg + nz) * plane]
    return bot_g, top_g, bot_i, top_i


class Comm:
    """Host hooks for one rank; subclasses implement allreduce / halo."""

    def __init__(self, nranks: int, rank: int, periodic: bool):
        self.nranks, self.rank, self.periodic = nranks, rank, periodic

    def lower(self):
        if self.rank > 0:
            return self.rank - 1
        return self.nranks - 1 if self.periodic else None

    def upper(self):
        if self.rank < self.nranks - 1:
            return self.rank + 1
        return 0 if self.periodic else None

    def allreduce(self, values: np.ndarray, op: str) -> None:
        raise NotImplementedError

    def halo(self, vec: torch.Tensor, plane: int, nz: int, zg: int, depth: int) -> None:
        raise NotImplementedError

    # ctypes trampolines handed to acch_set_comm ----------------------------
    def c_hooks(self, device):
        from . import _native as nat

        def _allreduce(user, values, n, op):
            try:
                arr = np.ctypeslib.as_array(values, shape=(n,))
                self.allreduce(arr, _OPS[op])
                return 0
            except Exception as e:  # surfaced through acch_last_error
                self.error = e
                return 1

        def _halo(user, vec, plane, nz, zg, depth):
            try:
                n = (nz + 2 * zg) * plane
                t = torch.as_tensor(_DevBuf(vec, n), device=device)
                self.halo(t, plane, nz, zg, depth)
                return 0
            except Exception as e:
                self.error = e
                return 1

        self._c_allreduce = nat.ALLREDUCE_FN(_allreduce)
        self._c_halo = nat.HALO_FN(_halo)
        return self._c_allreduce, self._c_halo


class TorchDistComm(Comm):
    """torch.distributed hooks (NCCL for CUDA tensors, gloo for CPU)."""

    def __init__(self, periodic: bool, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        super().__init__(dist.get_world_size(group), dist.get_rank(group), periodic)

    def allreduce(self, values: np.ndarray, op: str) -> None:
        dist = self.dist
        dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.as_tensor(values.copy(), device=dev)
        rop = {"sum": dist.ReduceOp.SUM, "min": dist.ReduceOp.MIN, "max": dist.ReduceOp.MAX}[op]
        dist.all_reduce(t, op=rop, group=self.group)
        values[:] = t.cpu().numpy()

    def halo(self, vec: torch.Tensor, plane: int, nz: int, zg: int, depth: int) -> None:
        dist = self.dist
        bot_g, top_g, bot_i, top_i = _ghost_views(vec, plane, nz, zg, depth)
        lo, hi = self.lower(), self.upper()
        if self.nranks == 1:
            if lo is not None:
                bot_g.copy_(top_i)
                top_g.copy_(bot_i)
            return
        recv_lo = torch.empty_like(bot_g) if lo is not None else None
        recv_hi = torch.empty_like(top_g) if hi is not None else None

        def peer(r):
            return dist.get_global_rank(self.group, r) if self.group is not None else r
        # per peer pair the sends go "up" first and the receives come "from
        # below" first, so two ranks that are each other's upper and lower
        # neighbour (2 periodic ranks) still match messages correctly
        ops = []
        if hi is not None:
            ops.append(dist.P2POp(dist.isend, top_i.contiguous(), peer(hi), self.group))
        if lo is not None:
            ops.append(dist.P2POp(dist.isend, bot_i.contiguous(), peer(lo), self.group))
        if lo is not None:
            ops.append(dist.P2POp(dist.irecv, recv_lo, peer(lo), self.group))
        if hi is not None:
            ops.append(dist.P2POp(dist.irecv, recv_hi, peer(hi), self.group))
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        if lo is not None:
            bot_g.copy_(recv_lo)
        if hi is not None:
            top_g.copy_(recv_hi)
        if vec.is_cuda:
            torch.cuda.current_stream(vec.device).synchronize()


def nccl_library_path() -> str | None:
    """The libnccl torch.distributed uses (its pip wheel), or None (then the
    library dlopens "libnccl.so.2", which resolves to the copy already loaded
    into the process)."""
    try:
        import nvidia.nccl
        import os
        base = list(nvidia.nccl.__path__)[0]
        path = os.path.join(base, "lib", "libnccl.so.2")
        return path if os.path.exists(path) else None
    except Exception:
        return None


class NcclComm(Comm):
    """The in-library NCCL data plane (csrc/comm.cu): every context on a slab
    grid bound to this communicator gets its own NCCL communicator, created
    collectively -- rank 0 draws an ncclUniqueId, torch.distributed
    broadcasts it (any backend: gloo on CPU works), every rank calls
    acch_set_nccl.  Halos and reductions then run as NCCL operations on the
    library's stream; nothing comes back to Python per exchange."""

    native = True

    def __init__(self, periodic: bool, group=None, nccl_path: str | None = None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.nccl_path = nccl_path if nccl_path is not None else nccl_library_path()
        super().__init__(dist.get_world_size(group), dist.get_rank(group), periodic)

    def unique_id(self) -> bytes:
        """A fresh ncclUniqueId, identical on every rank (collective)."""
        import ctypes
        from . import _native as nat
        L = nat.lib()
        nbytes = int(L.acch_nccl_id_bytes())
        buf = torch.zeros(nbytes, dtype=torch.uint8)
        if self.rank == 0:
            raw = (ctypes.c_char * nbytes)()
            path = self.nccl_path.encode() if self.nccl_path else None
            nat.check(L.acch_nccl_unique_id(path, raw), "acch_nccl_unique_id")
            buf.copy_(torch.frombuffer(bytearray(raw.raw), dtype=torch.uint8))
        dev_bcast = self.dist.get_backend(self.group) == "nccl"
        t = buf.cuda() if dev_bcast else buf
        src = self.dist.get_global_rank(self.group, 0) if self.group is not None else 0
        self.dist.broadcast(t, src=src, group=self.group)
        return bytes(t.cpu().numpy().tobytes())

    def bind(self, ctx_handle) -> None:
        """Collective: give the context its NCCL communicator."""
        import ctypes
        from . import _native as nat
        uid = self.unique_id()
        path = self.nccl_path.encode() if self.nccl_path else None
        nat.check(nat.lib().acch_set_nccl(ctx_handle, path, ctypes.c_char_p(uid), self.nranks, self.rank),
                  "acch_set_nccl")

    def allreduce(self, values: np.ndarray, op: str) -> None:   # pragma: no cover - the library reduces itself
        raise RuntimeError("NcclComm reduces inside the library")

    def halo(self, vec, plane, nz, zg, depth) -> None:           # pragma: no cover
        raise RuntimeError("NcclComm exchanges inside the library")


class ThreadGroup:
    """Shared state of ranks emulated as threads of one process."""

    def __init__(self, nranks: int):
        self.nranks = nranks
        self.barrier = threading.Barrier(nranks)
        self.slots = [None] * nranks

    def comm(self, rank: int, periodic: bool) -> "ThreadComm":
        return ThreadComm(self, rank, periodic)


class ThreadComm(Comm):
    """Collective hooks between threads of one process (see ThreadGroup)."""

    def __init__(self, group: ThreadGroup, rank: int, periodic: bool):
        super().__init__(group.nranks, rank, periodic)
        self.group = group

    def allreduce(self, values: np.ndarray, op: str) -> None:
        g = self.group
        g.slots[self.rank] = values.copy()
        g.barrier.wait()
        stack = np.stack(g.slots)
        g.barrier.wait()
        if op == "sum":
            # fixed rank order: the same result on every rank, every run
            acc = stack[0].copy()
            for r in range(1, self.nranks):
                acc = acc + stack[r]
        elif op == "min":
            acc = np.min(stack, axis=0)
        else:
            acc = np.max(stack, axis=0)
        values[:] = acc

    def halo(self, vec: torch.Tensor, plane: int, nz: int, zg: int, depth: int) -> None:
        g = self.group
        g.slots[self.rank] = vec
        g.barrier.wait()
        lo, hi = self.lower(), self.upper()
        bot_g, top_g, _, _ = _ghost_views(vec, plane, nz, zg, depth)
        if lo is not None:
            bot_g.copy_(_ghost_views(g.slots[lo], plane, nz, zg, depth)[3])
        if hi is not None:
            top_g.copy_(_ghost_views(g.slots[hi], plane, nz, zg, depth)[2])
        if vec.is_cuda:
            torch.cuda.current_stream(vec.device).synchronize()
        g.barrier.wait()


# ---------------------------------------------------------------------------
# registry: the communicator a slab grid's context uses
# ---------------------------------------------------------------------------

_comms: dict = {}


def bind_comm(slab: SlabGrid, comm: Comm) -> None:
    _comms[slab] = comm


def comm_for(slab: SlabGrid) -> Comm | None:
    return _comms.get(slab)


__all__ = ["SlabGrid", "split_grid", "local_fields", "Comm", "TorchDistComm", "NcclComm", "ThreadGroup",
           "ThreadComm", "bind_comm", "comm_for", "nccl_library_path"]
