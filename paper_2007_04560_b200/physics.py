"""Constitutive layer: parameters, the device state, admissibility, entropy
chord and the discrete energy (API of the reference's acch/physics.py:35-351).

All evaluations run in libacch_b200 kernels on the state's device.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .exceptions import DomainError, InadmissibleStateError
from .grid import Grid

#: physics.py:26
ADMISSIBILITY_MARGIN = 1e-12
#: physics.py:28-32
CHORD_BRANCH_FACTOR = 0.4


@dataclass(frozen=True)
class Params:
    """alpha, beta, gamma, theta, rho and the entropy series order (physics.py:35-58)."""

    alpha: float
    beta: float
    gamma: float
    theta: float
    rho: float
    series_order: int = 10

    def __post_init__(self):
        for name in ("alpha", "beta", "gamma", "theta", "rho"):
            if not (float(getattr(self, name)) > 0.0):
                raise ValueError(f"{name} must be strictly positive")
        if int(self.series_order) < 1:
            raise ValueError("series_order must be >= 1")
        if int(self.series_order) > 32:
            raise ValueError("series_order must be <= 32 on this backend")


DEFAULT_PARAMS = Params(alpha=4.0, beta=2.0, gamma=0.005, theta=0.1, rho=0.001)


class Field:
    """Device view of one scalar cell field (no ghost layer; grid.py:106-150)."""

    def __init__(self, grid: Grid, values: torch.Tensor):
        self.grid = grid
        self.values = values

    @property
    def interior(self) -> torch.Tensor:
        return self.values


def _default_device():
    nat.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def _as_device(a, device) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=torch.float64)
    return torch.as_tensor(np.asarray(a, dtype=float), device=device)


class State:
    """Pair (u, v) stored interleaved per cell on the device: ``x`` has shape
    (n_cells, 2), cells x-fastest, exactly the reference's solver-vector
    layout (scheme.py:58-66) so that ``x.view(-1)`` *is* the packed vector."""

    def __init__(self, grid: Grid, x: torch.Tensor):
        x = nat.dev_f64(x, 2 * grid.n_store, "state")
        self.grid = grid
        self.x = x.view(grid.n_store, 2)

    @classmethod
    def from_interior(cls, grid: Grid, u, v, device=None) -> "State":
        device = torch.device(device) if device is not None else (
            u.device if isinstance(u, torch.Tensor) and u.is_cuda else _default_device())
        if not isinstance(u, torch.Tensor) and not isinstance(v, torch.Tensor):
            u = np.asarray(u, dtype=float)
            v = np.asarray(v, dtype=float)
            if u.shape != grid.array_shape or v.shape != grid.array_shape:
                raise ValueError(f"interior shape {u.shape} does not match grid {grid.array_shape}")
            host = np.zeros((grid.n_store, 2))
            z0 = getattr(grid, "zoff", 0)
            host[z0:z0 + grid.n_cells, 0] = u.ravel()
            host[z0:z0 + grid.n_cells, 1] = v.ravel()
            return cls(grid, torch.from_numpy(host).to(device))
        ut = _as_device(u, device).reshape(-1)
        vt = _as_device(v, device).reshape(-1)
        if ut.numel() != grid.n_cells or vt.numel() != grid.n_cells:
            raise ValueError("interior shape does not match grid")
        x = torch.zeros((grid.n_store, 2), dtype=torch.float64, device=device)
        z0 = getattr(grid, "zoff", 0)
        x[z0:z0 + grid.n_cells, 0] = ut
        x[z0:z0 + grid.n_cells, 1] = vt
        return cls(grid, x)

    @property
    def device(self):
        return self.x.device

    @property
    def vector(self) -> torch.Tensor:
        """The packed 2N solver vector (a view, not a copy)."""
        return self.x.view(-1)

    def _interior(self):
        z0 = getattr(self.grid, "zoff", 0)
        return self.x[z0:z0 + self.grid.n_cells]

    @property
    def u(self) -> Field:
        return Field(self.grid, self._interior()[:, 0].view(self.grid.array_shape))

    @property
    def v(self) -> Field:
        return Field(self.grid, self._interior()[:, 1].view(self.grid.array_shape))

    def copy(self) -> "State":
        return State(self.grid, self.x.clone())

    def fill_ghosts(self) -> "State":
        """Ghosts are implicit (index arithmetic); kept for API parity."""
        return self

    def to_numpy(self):
        h = self._interior().detach().cpu().numpy()
        return h[:, 0].reshape(self.grid.array_shape).copy(), h[:, 1].reshape(self.grid.array_shape).copy()


def _ctx(grid: Grid, params: Params | None, device):
    return nat.context_for(grid, params or DEFAULT_PARAMS, device)


def state_gap(state: State) -> float:
    ctx = _ctx(state.grid, None, state.device)
    out = ctypes.c_double()
    nat.check(nat.lib().acch_admissibility_gap(ctx.bind(), nat.ptr(state.x), ctypes.byref(out)), "gap")
    return out.value


def admissibility_gap(u, v=None) -> float:
    """Smallest distance from the admissible-set boundary (physics.py:89-109).
    Accepts a State or a (u, v) pair of arrays/tensors."""
    if isinstance(u, State):
        return state_gap(u)
    if v is None:
        raise TypeError("admissibility_gap takes a State or a (u, v) pair")
    nat.require_cuda()
    dev = u.device if isinstance(u, torch.Tensor) and u.is_cuda else (
        v.device if isinstance(v, torch.Tensor) and v.is_cuda else _default_device())
    ut, vt = torch.broadcast_tensors(_as_device(u, dev), _as_device(v, dev))
    if ut.numel() == 0:
        raise ValueError("admissibility_gap of an empty field")
    x = torch.stack((ut.reshape(-1), vt.reshape(-1)), dim=1).contiguous()
    from .grid import BoundaryCondition
    ctx = _ctx(Grid((4, 4), (1.0, 1.0), BoundaryCondition.PERIODIC), None, dev)
    out = ctypes.c_double()
    nat.check(nat.lib().acch_gap_pairs(ctx.bind(), nat.ptr(x), ut.numel(), ctypes.byref(out)), "gap_pairs")
    return out.value


def is_admissible(state: State, margin: float = ADMISSIBILITY_MARGIN) -> bool:
    return state_gap(state) >= margin


def check_admissible(state: State, margin: float = ADMISSIBILITY_MARGIN) -> None:
    gap = state_gap(state)
    if not gap >= margin:
        raise InadmissibleStateError(
            f"state violates admissibility bounds (gap {gap:.3e} < margin {margin:.1e})")


def _chord(a, b, order, force_exact, want_deriv):
    nat.require_cuda()
    scalar = np.ndim(a) == 0 and np.ndim(b) == 0 and not isinstance(a, torch.Tensor)
    dev = a.device if isinstance(a, torch.Tensor) and a.is_cuda else _default_device()
    at = _as_device(a, dev)
    bt = _as_device(b, dev)
    at, bt = torch.broadcast_tensors(at, bt)
    at = at.contiguous()
    bt = bt.contiguous()
    lo = min(float(at.min()), float(bt.min())) if at.numel() else 0.5
    hi = max(float(at.max()), float(bt.max())) if at.numel() else 0.5
    if not (lo > 0.0 and hi < 1.0):
        raise DomainError("entropy chord arguments must lie strictly inside (0, 1)")
    val = torch.empty_like(at)
    der = torch.empty_like(at) if want_deriv else None
    from .grid import BoundaryCondition
    g = Grid((4, 4), (1.0, 1.0), BoundaryCondition.PERIODIC)
    p = Params(4.0, 2.0, 0.005, 0.1, 0.001, int(order))
    ctx = _ctx(g, p, dev)
    nat.check(nat.lib().acch_entropy_chord(ctx.bind(), nat.ptr(at), nat.ptr(bt), at.numel(), int(bool(force_exact)),
                                           nat.ptr(val), nat.ptr(der) if der is not None else None), "chord")
    if scalar:
        return (float(val), float(der)) if want_deriv else float(val)
    return (val, der) if want_deriv else val


def entropy_chord(a, b, order: int = 10, force_exact: bool = False):
    """(Phi(a) - Phi(b)) / (a - b) with the reference's exact / series /
    direct branches (physics.py:213-262), evaluated on the device."""
    return _chord(a, b, order, force_exact, False)


def entropy_chord_with_deriv(a, b, order: int = 10, force_exact: bool = False):
    """Chord and its derivative in the first argument (physics.py:265-310)."""
    return _chord(a, b, order, force_exact, True)


def diagnostics(state: State, params: Params):
    """(total energy, integrate(u), max|v|) in one fused device reduction
    (physics.py:325-331, grid.py:301-303, cli/drivers.py:62-73)."""
    ctx = _ctx(state.grid, params, state.device)
    e, m, v = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    nat.check(nat.lib().acch_diagnostics(ctx.bind(), nat.ptr(state.x), ctypes.byref(e), ctypes.byref(m),
                                         ctypes.byref(v)), "diagnostics")
    return e.value, m.value, v.value


def total_energy(state: State, params: Params) -> float:
    """Discrete total free energy <e> (physics.py:325-331)."""
    return diagnostics(state, params)[0]


def integrate_u(state: State) -> float:
    return diagnostics(state, DEFAULT_PARAMS)[1]


__all__ = ["ADMISSIBILITY_MARGIN", "CHORD_BRANCH_FACTOR", "Params", "State", "Field", "admissibility_gap",
           "is_admissible", "check_admissible", "entropy_chord", "entropy_chord_with_deriv", "total_energy",
           "diagnostics"]
