"""ctypes binding of libacch_b200.so (the C ABI in include/acch_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
sm_100a) and lives next to this file.  There is no fallback: importing a
solver entry point without the library, or without a CUDA device, raises.
PyTorch is used only to own device buffers and to supply the current stream.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

from .exceptions import (InadmissibleStateError, PartitionError, ZeroPivotError)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ACCH_LIB_PATH") or os.path.join(_HERE, "libacch_b200.so")   # override: experiments only

ACCH_OK = 0
ACCH_ERR_INVALID_ARG = 1
ACCH_ERR_INADMISSIBLE = 2
ACCH_ERR_ZERO_PIVOT = 3
ACCH_ERR_CUDA = 4
ACCH_ERR_NO_FACTOR = 5
ACCH_ERR_PARTITION = 6


class GridDesc(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("periodic", ctypes.c_int32),
                ("counts", ctypes.c_int64 * 3), ("lengths", ctypes.c_double * 3)]


class ParamsDesc(ctypes.Structure):
    _fields_ = [("alpha", ctypes.c_double), ("beta", ctypes.c_double), ("gamma", ctypes.c_double),
                ("theta", ctypes.c_double), ("rho", ctypes.c_double), ("series_order", ctypes.c_int32)]


class SlabDesc(ctypes.Structure):
    _fields_ = [("nranks", ctypes.c_int32), ("rank", ctypes.c_int32), ("ghost_planes", ctypes.c_int32),
                ("wall_lo", ctypes.c_int32), ("wall_hi", ctypes.c_int32), ("z_offset", ctypes.c_int32),
                ("nz_global", ctypes.c_int32)]


ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.c_int32,
                                ctypes.c_int32)
HALO_FN = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                           ctypes.c_int32, ctypes.c_int32)

_P = ctypes.c_void_p
_D = ctypes.c_double
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_PD = ctypes.POINTER(ctypes.c_double)
_PI32 = ctypes.POINTER(ctypes.c_int32)
_PI64 = ctypes.POINTER(ctypes.c_int64)

# name -> (restype, argtypes); the exported surface of include/acch_b200.h
SIGNATURES = {
    "acch_last_error": (ctypes.c_char_p, []),
    "acch_abi_version": (_I32, []),
    "acch_ctx_create": (_I32, [ctypes.POINTER(GridDesc), ctypes.POINTER(ParamsDesc), _I32, ctypes.POINTER(_P)]),
    "acch_ctx_destroy": (_I32, [_P]),
    "acch_set_stream": (_I32, [_P, _P]),
    "acch_entropy_chord": (_I32, [_P, _P, _P, _I64, _I32, _P, _P]),
    "acch_admissibility_gap": (_I32, [_P, _P, _PD]),
    "acch_gap_pairs": (_I32, [_P, _P, _I64, _PD]),
    "acch_diagnostics": (_I32, [_P, _P, _PD, _PD, _PD]),
    "acch_residual": (_I32, [_P, _P, _D, _P, _P, _PD, _PD]),
    "acch_jacobian_prepare": (_I32, [_P, _P, _D, _P, _P]),
    "acch_jacobian_matvec": (_I32, [_P, _P, _D, _P, _P]),
    "acch_jacobian_blocks": (_I32, [_P, _P, _D, _P]),
    "acch_stencil_offsets": (_I32, [_I32, _PI32]),
    "acch_dot": (_I32, [_P, _P, _P, _I64, _PD]),
    "acch_rms_diff": (_I32, [_P, _P, _P, _I64, _PD]),
    "acch_axpby": (_I32, [_P, _D, _P, _D, _P, _I64]),
    "acch_trial": (_I32, [_P, _P, _P, _D, _P, _PD]),
    "acch_feasible_cap": (_I32, [_P, _P, _P, _D, _D, _PD]),
    "acch_precond_create": (_I32, [_P, _I64, _I32, _PI64, _PI64, _I32, _I32, ctypes.POINTER(_P)]),
    "acch_precond_destroy": (_I32, [_P]),
    "acch_precond_update": (_I32, [_P, _P, _D, _I32, _PI32, _PI64, _PI32]),
    "acch_precond_invalidate": (_I32, [_P]),
    "acch_precond_apply": (_I32, [_P, _P, _P]),
    "acch_precond_info": (_I32, [_P, _PI64, _PI64, _PI64]),
    "acch_gmres": (_I32, [_P, _P, _D, _P, _P, _P, _D, _D, _I32, _I32, _I32, _PI32, _PI32, _PD]),
    "acch_gmres_x0": (_I32, [_P, _P, _D, _P, _P, _P, _I32, _D, _D, _I32, _I32, _I32, _PI32, _PI32, _PD]),
    "acch_launch_count": (_I64, [_P]),
    "acch_profile_enable": (_I32, [_P, _I32]),
    "acch_ctx_set_slab": (_I32, [_P, ctypes.POINTER(SlabDesc)]),
    "acch_set_comm": (_I32, [_P, ALLREDUCE_FN, HALO_FN, _P]),
    "acch_storage_cells": (_I64, [_P]),
    "acch_profile_read": (_I32, [_P, _PD, _PI64, _PD, _I32]),
    "acch_nccl_unique_id": (_I32, [ctypes.c_char_p, ctypes.c_void_p]),
    "acch_nccl_id_bytes": (_I32, []),
    "acch_set_nccl": (_I32, [_P, ctypes.c_char_p, ctypes.c_char_p, _I32, _I32]),
    "acch_comm_stats": (_I32, [_P, _PD, _PI64]),
}

PROFILE_CATEGORIES = ("residual", "jacobian_prepare", "matvec", "precond_factor", "precond_apply",
                      "precond_gather", "krylov_dot", "krylov_update", "krylov_vector", "state_reductions")

_lib = None
_lock = threading.Lock()


def load_library(path: str = LIB_PATH):
    """Load and bind libacch_b200.so (no GPU needed to load)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise ImportError(
                    f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(nvcc, sm_100a).  There is no CPU fallback.")
            lib = ctypes.CDLL(path)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def lib():
    return load_library()


def last_error() -> str:
    msg = lib().acch_last_error()
    return msg.decode() if msg else ""


class NativeError(RuntimeError):
    pass


def check(status: int, what: str = ""):
    """Map an acch_status onto the reference's exception classes."""
    if status == ACCH_OK:
        return
    msg = last_error()
    if status == ACCH_ERR_INADMISSIBLE:
        raise InadmissibleStateError(msg)
    if status == ACCH_ERR_PARTITION:
        raise PartitionError(msg)
    if status == ACCH_ERR_INVALID_ARG:
        raise ValueError(f"{what}: {msg}")
    if status == ACCH_ERR_NO_FACTOR:
        raise RuntimeError(msg)
    raise NativeError(f"{what}: {msg} (status {status})")


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2007_04560_b200 needs a CUDA device (B200, sm_100a); there is no CPU path")


def ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


def dev_f64(t: torch.Tensor, n: int | None = None, name: str = "tensor") -> torch.Tensor:
    """Validate a solver buffer: contiguous fp64 on a CUDA device."""
    if not isinstance(t, torch.Tensor) or t.device.type != "cuda" or t.dtype != torch.float64:
        raise TypeError(f"{name} must be a float64 CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if n is not None and t.numel() != n:
        raise ValueError(f"{name} has {t.numel()} entries, expected {n}")
    return t


class Context:
    """Owns one acch_ctx (grid + params + reduction scratch + Krylov space)."""

    def __init__(self, grid, params, device: torch.device):
        require_cuda()
        self.grid = grid
        self.params = params
        self.device = torch.device(device)
        desc = GridDesc()
        desc.dim = grid.dim
        desc.periodic = 1 if grid.periodic else 0
        for a in range(3):
            desc.counts[a] = grid.counts[a] if a < grid.dim else 1
            desc.lengths[a] = grid.lengths[a] if a < grid.dim else 1.0
        pd = ParamsDesc(params.alpha, params.beta, params.gamma, params.theta, params.rho,
                        int(params.series_order))
        h = _P()
        idx = self.device.index if self.device.index is not None else torch.cuda.current_device()
        check(lib().acch_ctx_create(ctypes.byref(desc), ctypes.byref(pd), idx, ctypes.byref(h)),
              "acch_ctx_create")
        self.handle = h
        self._lib = lib()
        self.comm = None
        if getattr(grid, "nz_global", 0):
            # a z-slab of a decomposed grid: ghost planes + cross-rank hooks
            from .slab import comm_for
            sd = SlabDesc(grid.nranks, grid.rank, grid.ghost, int(grid.wall_lo), int(grid.wall_hi), grid.z0,
                          grid.nz_global)
            check(self._lib.acch_ctx_set_slab(h, ctypes.byref(sd)), "acch_ctx_set_slab")
            comm = comm_for(grid)
            if comm is None:
                raise RuntimeError("no communicator bound to this slab grid (slab.bind_comm)")
            if getattr(comm, "native", False):
                comm.bind(h)            # in-library NCCL (collective across ranks)
            else:
                ar, ha = comm.c_hooks(self.device)
                check(self._lib.acch_set_comm(h, ar, ha, None), "acch_set_comm")
            self.comm = comm

    def bind(self):
        """Point the context at the current torch stream; returns the handle."""
        s = torch.cuda.current_stream(self.device).cuda_stream
        self._lib.acch_set_stream(self.handle, _P(s))
        return self.handle

    @property
    def launches(self) -> int:
        return int(self._lib.acch_launch_count(self.handle))

    def comm_stats(self) -> dict:
        """Halo bytes sent and NCCL calls made by this context."""
        b, c = ctypes.c_double(), ctypes.c_int64()
        check(self._lib.acch_comm_stats(self.handle, ctypes.byref(b), ctypes.byref(c)), "comm_stats")
        return {"halo_bytes": b.value, "nccl_calls": c.value}

    def profile(self, on: bool = True):
        check(self._lib.acch_profile_enable(self.handle, int(bool(on))), "profile_enable")

    def profile_read(self) -> dict:
        """{category: (milliseconds, launches, algorithmic bytes)} since the last read."""
        n = len(PROFILE_CATEGORIES)
        ms = (ctypes.c_double * n)()
        cnt = (ctypes.c_int64 * n)()
        nb = (ctypes.c_double * n)()
        self.bind()
        check(self._lib.acch_profile_read(self.handle, ms, cnt, nb, n), "profile_read")
        return {k: (ms[i], cnt[i], nb[i]) for i, k in enumerate(PROFILE_CATEGORIES)}

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _lib is not None:
            try:
                _lib.acch_ctx_destroy(h)
            except Exception:
                pass
            self.handle = None


_contexts: dict = {}


def context_for(grid, params, device=None) -> Context:
    """One native context per (grid, params, device), like the reference's
    lru-cached grid operators (scheme.py:166-167)."""
    require_cuda()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    key = (grid, params, dev.index)
    ctx = _contexts.get(key)
    if ctx is None:
        ctx = Context(grid, params, dev)
        _contexts[key] = ctx
    return ctx


def total_launches() -> int:
    return sum(c.launches for c in _contexts.values())
