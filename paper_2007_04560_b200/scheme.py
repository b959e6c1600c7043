"""The implicit energy-stable step: residual and Jacobian (API of the
reference's acch/scheme.py:58-498), backed by the fused sm_100a kernels.

* ``residual_vector`` -> one fused stencil kernel (acch_residual) that also
  returns ||F||^2 and the admissibility gap of the iterate.
* ``assemble_jacobian`` -> a JacobianOperator: 7 coefficient planes
  (acch_jacobian_prepare) plus a matrix-free radius-2 matvec
  (acch_jacobian_matvec).  The reference assembles a 2x2-block BSR matrix
  (scheme.py:427-484); the same blocks are available on demand
  (``JacobianOperator.blocks`` / ``to_bsr``) and the Schwarz factorisation
  builds its subdomain rows from the planes directly.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as nat
from .grid import Grid
from .physics import ADMISSIBILITY_MARGIN, Params, State, check_admissible

N_COEF = 7   # S, D, cbar, G_u, c_u, c_v, G_v


# ---------------------------------------------------------------------------
# vector packing (interleaved u, v per cell, x fastest; scheme.py:58-80)
# ---------------------------------------------------------------------------

def pack_fields(u, v) -> torch.Tensor:
    """Interleave two cell fields into the 2N solver vector."""
    ut = u if isinstance(u, torch.Tensor) else torch.as_tensor(np.asarray(u, dtype=float))
    vt = v if isinstance(v, torch.Tensor) else torch.as_tensor(np.asarray(v, dtype=float))
    return torch.stack([ut.reshape(-1), vt.reshape(-1)], dim=1).reshape(-1)


def unpack_vector(grid: Grid, x: torch.Tensor):
    """Views of the u and v components of a packed vector."""
    x2 = x.view(grid.n_store, 2)
    z0 = getattr(grid, "zoff", 0)
    x2 = x2[z0:z0 + grid.n_cells]
    return x2[:, 0].view(grid.array_shape), x2[:, 1].view(grid.array_shape)


def vector_from_state(state: State) -> torch.Tensor:
    return state.vector.clone()


def state_from_vector(grid: Grid, x: torch.Tensor) -> State:
    return State(grid, x.clone() if isinstance(x, torch.Tensor) else torch.as_tensor(x))


def trial_state(grid: Grid, base: torch.Tensor, direction: torch.Tensor, step: float) -> State:
    """State at base + step * direction (scheme.py:487-498); may be inadmissible."""
    ctx = nat.context_for(grid, _GRID_ONLY_PARAMS, base.device)
    out = torch.empty_like(base)
    gap = ctypes.c_double()
    nat.check(nat.lib().acch_trial(ctx.bind(), nat.ptr(base), nat.ptr(direction), float(step), nat.ptr(out),
                                   ctypes.byref(gap)), "trial")
    st = State(grid, out)
    st._gap = gap.value
    return st


_GRID_ONLY_PARAMS = Params(4.0, 2.0, 0.005, 0.1, 0.001)


# ---------------------------------------------------------------------------
# one implicit time step
# ---------------------------------------------------------------------------

@dataclass
class StepProblem:
    """Frozen data of one implicit step: old state and dt (scheme.py:195-267).

    The old state is copied into a device buffer owned by the problem; the
    old-level mobility and Laplacians the reference caches (scheme.py:234-246)
    are recomputed inside the fused kernels instead of being stored."""

    grid: Grid
    params: Params
    old: State
    dt: float
    _ctx: object = field(default=None, repr=False)

    @classmethod
    def create(cls, grid: Grid, params: Params, old: State, dt: float) -> "StepProblem":
        if not dt > 0.0:
            raise ValueError("time step must be positive")
        check_admissible(old)
        ctx = nat.context_for(grid, params, old.device)
        return cls(grid, params, old.copy(), float(dt), ctx)

    @property
    def ctx(self):
        return self._ctx

    def residual_into(self, x: torch.Tensor, out: torch.Tensor):
        """F(x) into ``out``; returns (||F||_2, gap).  Raises
        InadmissibleStateError like check_admissible (scheme.py:250)."""
        gap, n2 = ctypes.c_double(), ctypes.c_double()
        nat.check(nat.lib().acch_residual(self._ctx.bind(), nat.ptr(self.old.x), self.dt, nat.ptr(x), nat.ptr(out),
                                          ctypes.byref(gap), ctypes.byref(n2)), "residual")
        return math.sqrt(n2.value), gap.value


def _vec(state_or_vec, grid: Grid) -> torch.Tensor:
    if isinstance(state_or_vec, State):
        return state_or_vec.vector
    return nat.dev_f64(state_or_vec, 2 * grid.n_store, "vector")


def residual_vector(prob: StepProblem, new) -> torch.Tensor:
    """Packed residual F(new) of the implicit step (scheme.py:343-354)."""
    x = _vec(new, prob.grid)
    out = torch.empty_like(x)
    prob.residual_into(x, out)
    return out


def step_residual(prob: StepProblem, new):
    """(F_u, F_v) as cell-field views (scheme.py:343-349)."""
    return unpack_vector(prob.grid, residual_vector(prob, new))


class JacobianOperator:
    """Analytic Jacobian of the step residual at one iterate, matrix-free.

    ``matvec`` applies exactly the operator scheme.py:471-482 assembles
    (2x2 blocks on the radius-2 skeleton), from 7 per-cell coefficient planes."""

    def __init__(self, prob: StepProblem, coef: torch.Tensor):
        self.prob = prob
        self.grid = prob.grid
        self.coef = coef
        self.dt = prob.dt
        self.n_cells = prob.grid.n_cells
        self.n_store = prob.grid.n_store

    @property
    def shape(self):
        return (2 * self.n_cells, 2 * self.n_cells)

    @property
    def ctx(self):
        return self.prob.ctx

    def matvec_into(self, w: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
        nat.check(nat.lib().acch_jacobian_matvec(self.ctx.bind(), nat.ptr(self.coef), self.dt, nat.ptr(w), nat.ptr(y)),
                  "matvec")
        return y

    def matvec(self, w) -> torch.Tensor:
        w = nat.dev_f64(w if isinstance(w, torch.Tensor) else torch.as_tensor(w, device=self.coef.device),
                        2 * self.n_store, "w")
        return self.matvec_into(w, torch.empty_like(w))

    __call__ = matvec

    def blocks(self) -> torch.Tensor:
        """Stencil blocks: (N, n_offsets, 2, 2) with offsets ``stencil_offsets``."""
        noff = nat.lib().acch_stencil_offsets(self.grid.dim, None)
        out = torch.empty((self.n_cells, noff, 2, 2), dtype=torch.float64, device=self.coef.device)
        nat.check(nat.lib().acch_jacobian_blocks(self.ctx.bind(), nat.ptr(self.coef), self.dt, nat.ptr(out)),
                  "jacobian_blocks")
        return out

    def to_bsr(self):
        """Host scipy BSR on the reference's skeleton (scheme.py:166-188):
        duplicate stencil targets (periodic axes of 4 cells) are summed and
        offsets leaving a Neumann box are dropped."""
        from scipy import sparse
        blocks = self.blocks().cpu().numpy()
        offs = stencil_offsets(self.grid.dim)
        g = self.grid
        n = g.n_cells
        ids = np.arange(n)
        coords = [ids % g.counts[0], (ids // g.counts[0]) % g.counts[1]]
        if g.dim == 3:
            coords.append(ids // (g.counts[0] * g.counts[1]))
        rows, cols, vals = [], [], []
        for q, off in enumerate(offs):
            ok = np.ones(n, dtype=bool)
            tgt = np.zeros(n, dtype=np.int64)
            stride = 1
            for a in range(g.dim):
                t = coords[a] + off[a]
                if g.periodic:
                    t = t % g.counts[a]
                else:
                    ok &= (t >= 0) & (t < g.counts[a])
                tgt += np.clip(t, 0, g.counts[a] - 1) * stride
                stride *= g.counts[a]
            rows.append(ids[ok])
            cols.append(tgt[ok])
            vals.append(blocks[ok, q])
        rows = np.concatenate(rows)
        cols = np.concatenate(cols)
        vals = np.concatenate(vals)
        r2 = np.concatenate([2 * rows, 2 * rows, 2 * rows + 1, 2 * rows + 1])
        c2 = np.concatenate([2 * cols, 2 * cols + 1, 2 * cols, 2 * cols + 1])
        v2 = np.concatenate([vals[:, 0, 0], vals[:, 0, 1], vals[:, 1, 0], vals[:, 1, 1]])
        csr = sparse.coo_matrix((v2, (r2, c2)), shape=(2 * n, 2 * n)).tocsr()
        csr.sum_duplicates()
        return csr.tobsr(blocksize=(2, 2))


def stencil_offsets(dim: int):
    buf = (ctypes.c_int32 * 75)()
    n = nat.lib().acch_stencil_offsets(dim, buf)
    return [(buf[3 * i], buf[3 * i + 1], buf[3 * i + 2]) for i in range(n)]


def assemble_jacobian(prob: StepProblem, new) -> JacobianOperator:
    """Jacobian of the step residual at ``new`` (scheme.py:427-484)."""
    x = _vec(new, prob.grid)
    coef = torch.empty(N_COEF * prob.grid.n_store, dtype=torch.float64, device=x.device)
    gap = ctypes.c_double()
    nat.check(nat.lib().acch_admissibility_gap(prob.ctx.bind(), nat.ptr(x), ctypes.byref(gap)), "gap")
    if not gap.value >= ADMISSIBILITY_MARGIN:
        from .exceptions import InadmissibleStateError
        raise InadmissibleStateError(f"state violates admissibility bounds (gap {gap.value:.3e})")
    nat.check(nat.lib().acch_jacobian_prepare(prob.ctx.bind(), nat.ptr(prob.old.x), prob.dt, nat.ptr(x),
                                              nat.ptr(coef)), "jacobian_prepare")
    return JacobianOperator(prob, coef)


def prepare_jacobian_unchecked(prob: StepProblem, x: torch.Tensor, coef: torch.Tensor) -> JacobianOperator:
    """assemble_jacobian for an iterate already known to be admissible (the
    Newton loop's accepted iterate); skips the extra gap reduction."""
    nat.check(nat.lib().acch_jacobian_prepare(prob.ctx.bind(), nat.ptr(prob.old.x), prob.dt, nat.ptr(x),
                                              nat.ptr(coef)), "jacobian_prepare")
    return JacobianOperator(prob, coef)
