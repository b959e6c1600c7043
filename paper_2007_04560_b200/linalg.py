"""Domain decomposition, the Schwarz preconditioner and GMRES (API of the
reference's acch/linalg.py:112-506).

``partition`` runs on the host (once per run, numpy) and reproduces the
reference's boxes, ordering and extension exactly.  The preconditioner's
symbolic analysis (box classes, ILU fill patterns, level schedules) is native
C++ inside libacch_b200; factorisation and applies are CUDA kernels, one CTA
per subdomain.  ``gmres`` with a JacobianOperator runs the restarted GMRES
driver inside the library (device vectors, host Hessenberg)."""

from __future__ import annotations

import ctypes
import enum
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as nat
from .exceptions import PartitionError, ZeroPivotError
from .grid import BoundaryCondition, Grid

BLOCK = 2


# ---------------------------------------------------------------------------
# domain decomposition (linalg.py:112-210)
# ---------------------------------------------------------------------------

def _factor_tuples(n: int, dims: int):
    if dims == 1:
        yield (n,)
        return
    for d in range(1, n + 1):
        if n % d == 0:
            for rest in _factor_tuples(n // d, dims - 1):
                yield (d,) + rest


@dataclass
class Decomposition:
    """Overlapping Cartesian decomposition (linalg.py:112-121).

    ``owned_lo`` / ``owned_hi`` ([n_sub, 3]) are the owned cell ranges per
    axis that the native preconditioner consumes; the reference's per-box id
    arrays are materialised lazily on first access."""

    grid: Grid
    n_subdomains: int
    overlap: int
    factors: tuple
    owned_lo: np.ndarray
    owned_hi: np.ndarray
    _cache: dict = field(default_factory=dict, repr=False)

    def _axis_ext(self, a, lo, hi):
        n = self.grid.counts[a]
        if self.grid.periodic:
            return np.unique(np.arange(lo - self.overlap, hi + self.overlap) % n).astype(np.int64)
        return np.arange(max(lo - self.overlap, 0), min(hi + self.overlap, n), dtype=np.int64)

    def _flat(self, axes):
        c = self.grid.counts
        if self.grid.dim == 2:
            ix, iy = axes
            return (iy[:, None] * c[0] + ix[None, :]).ravel()
        ix, iy, iz = axes
        return ((iz[:, None, None] * c[1] + iy[None, :, None]) * c[0] + ix[None, None, :]).ravel()

    def _build(self):
        own, ext, pos = [], [], []
        for s in range(self.n_subdomains):
            oa = [np.arange(self.owned_lo[s, a], self.owned_hi[s, a], dtype=np.int64) for a in range(self.grid.dim)]
            ea = [self._axis_ext(a, self.owned_lo[s, a], self.owned_hi[s, a]) for a in range(self.grid.dim)]
            o = self._flat(oa)
            e = self._flat(ea)
            own.append(o)
            ext.append(e)
            pos.append(np.searchsorted(e, o))
        self._cache.update(owned=own, extended=ext, pos=pos)

    @property
    def owned_cells(self):
        if "owned" not in self._cache:
            self._build()
        return self._cache["owned"]

    @property
    def extended_cells(self):
        if "extended" not in self._cache:
            self._build()
        return self._cache["extended"]

    @property
    def owned_in_extended(self):
        if "pos" not in self._cache:
            self._build()
        return self._cache["pos"]


def partition(grid: Grid, n_subdomains: int, overlap: int) -> Decomposition:
    """Near-cubical boxes, ties broken lexicographically, remainder cells to
    the first boxes, boxes ordered z slowest (linalg.py:161-210)."""
    if n_subdomains < 1:
        raise PartitionError("need at least one subdomain")
    if overlap < 0:
        raise PartitionError("overlap must be nonnegative")
    if getattr(grid, "nz_global", 0):
        return _slab_partition(grid, n_subdomains, overlap)
    best = None
    for f in _factor_tuples(int(n_subdomains), grid.dim):
        if any(f[a] > grid.counts[a] for a in range(grid.dim)):
            continue
        edges = [grid.counts[a] / f[a] for a in range(grid.dim)]
        key = (max(edges) / min(edges), f)
        if best is None or key < best:
            best = key
    if best is None:
        raise PartitionError(f"cannot split {grid.counts} into {n_subdomains} boxes of at least one cell")
    factors = best[1]
    bounds = []
    for a in range(grid.dim):
        n, p = grid.counts[a], factors[a]
        sizes = np.full(p, n // p, dtype=np.int64)
        sizes[: n % p] += 1
        ends = np.cumsum(sizes)
        bounds.append((ends - sizes, ends))
    lo = np.zeros((n_subdomains, 3), dtype=np.int64)
    hi = np.ones((n_subdomains, 3), dtype=np.int64)
    for s, rev in enumerate(np.ndindex(*reversed(factors))):
        idx = tuple(reversed(rev))
        for a in range(grid.dim):
            lo[s, a] = bounds[a][0][idx[a]]
            hi[s, a] = bounds[a][1][idx[a]]
    return Decomposition(grid, int(n_subdomains), int(overlap), tuple(factors), lo, hi)


def _slab_partition(slab, n_subdomains: int, overlap: int) -> Decomposition:
    """The global partition's boxes that lie in this rank's z-slab, in local
    z coordinates (box order kept).  Slab boundaries must fall on box
    boundaries, so every global box belongs to exactly one rank."""
    glob = partition(slab.global_grid(), n_subdomains, overlap)
    z0, z1 = slab.z0, slab.z0 + slab.counts[2]
    zl, zh = glob.owned_lo[:, 2], glob.owned_hi[:, 2]
    inside = (zl >= z0) & (zh <= z1)
    straddle = (zl < z1) & (zh > z0) & ~inside
    if straddle.any():
        raise PartitionError(f"box z-ranges do not align with the slab [{z0}, {z1}) of rank {slab.rank}")
    lo = glob.owned_lo[inside].copy()
    hi = glob.owned_hi[inside].copy()
    lo[:, 2] -= z0
    hi[:, 2] -= z0
    return Decomposition(slab, int(inside.sum()), int(overlap), glob.factors, lo, hi)


# ---------------------------------------------------------------------------
# Schwarz preconditioner (linalg.py:217-396)
# ---------------------------------------------------------------------------

class SchwarzVariant(enum.Enum):
    CLASSICAL = "asm"
    LEFT_RAS = "ras-left"
    RIGHT_RAS = "ras-right"


_VARIANT_CODE = {SchwarzVariant.CLASSICAL: 0, SchwarzVariant.LEFT_RAS: 1, SchwarzVariant.RIGHT_RAS: 2}


@dataclass(frozen=True)
class SubdomainSolverSpec:
    """ILU with a fill level, or exact LU (linalg.py:224-246)."""

    kind: str
    fill_level: int = 0

    def __post_init__(self):
        if self.kind not in ("ilu", "lu"):
            raise ValueError(f"unknown subdomain solver kind {self.kind!r}")
        if self.kind == "ilu" and self.fill_level < 0:
            raise ValueError("fill level must be nonnegative")

    @classmethod
    def from_string(cls, text: str) -> "SubdomainSolverSpec":
        text = text.strip().lower()
        if text == "lu":
            return cls("lu")
        if text.startswith("ilu") and text[3:].isdigit():
            return cls("ilu", int(text[3:]))
        raise ValueError(f"unknown subdomain solver {text!r} (use ilu0/ilu1/ilu2/lu)")

    def __str__(self):
        return "lu" if self.kind == "lu" else f"ilu{self.fill_level}"


class SchwarzPreconditioner:
    """ASM / left-RAS / right-RAS with ILU(k) or exact-LU subdomain solves
    (linalg.py:320-396).  ``pool`` is accepted for API parity; the GPU runs
    all subdomains concurrently (one CTA each).

    The "lu" subdomain solver is a complete (no-drop) factorisation in the
    reference's local ordering without pivoting: the exact subdomain solve,
    as SuperLU computes it up to rounding."""

    def __init__(self, decomposition: Decomposition, variant: SchwarzVariant,
                 subsolver: SubdomainSolverSpec, pool=None):
        self.decomposition = decomposition
        self.variant = SchwarzVariant(variant)
        self.subsolver = subsolver
        self.pool = pool
        self._handle = None
        self._ctx = None
        self.factorization_count = 0

    def _ensure(self, ctx):
        if self._handle is not None:
            if ctx is not self._ctx:
                raise ValueError("preconditioner is bound to another grid/params context")
            return
        d = self.decomposition
        lo = np.ascontiguousarray(d.owned_lo, dtype=np.int64)
        hi = np.ascontiguousarray(d.owned_hi, dtype=np.int64)
        fill = -1 if self.subsolver.kind == "lu" else int(self.subsolver.fill_level)
        h = ctypes.c_void_p()
        p64 = ctypes.POINTER(ctypes.c_int64)
        nat.check(nat.lib().acch_precond_create(ctx.bind(), d.n_subdomains, d.overlap, lo.ctypes.data_as(p64),
                                                hi.ctypes.data_as(p64), _VARIANT_CODE[self.variant], fill,
                                                ctypes.byref(h)), "precond_create")
        self._handle = h
        self._ctx = ctx

    def invalidate(self) -> None:
        if self._handle is not None:
            nat.check(nat.lib().acch_precond_invalidate(self._handle), "precond_invalidate")

    @property
    def handle(self):
        return self._handle

    def update(self, matrix, reuse: bool = False) -> bool:
        """(Re)factor from a JacobianOperator; with reuse keep valid factors.
        Returns True when a factorisation happened (linalg.py:353-372)."""
        self._ensure(matrix.ctx)
        ref = ctypes.c_int32()
        cell = ctypes.c_int64()
        comp = ctypes.c_int32()
        st = nat.lib().acch_precond_update(self._handle, nat.ptr(matrix.coef), matrix.dt, int(bool(reuse)),
                                           ctypes.byref(ref), ctypes.byref(cell), ctypes.byref(comp))
        if st == nat.ACCH_ERR_ZERO_PIVOT:
            self.factorization_count += 1
            raise ZeroPivotError(int(cell.value), int(comp.value))
        nat.check(st, "precond_update")
        if ref.value:
            self.factorization_count += 1
        return bool(ref.value)

    def apply_into(self, r: torch.Tensor, z: torch.Tensor) -> torch.Tensor:
        if self._handle is None:
            raise RuntimeError("preconditioner has no factorization; call update() first")
        self._ctx.bind()
        nat.check(nat.lib().acch_precond_apply(self._handle, nat.ptr(r), nat.ptr(z)), "precond_apply")
        return z

    def apply(self, r) -> torch.Tensor:
        if not isinstance(r, torch.Tensor):
            r = torch.as_tensor(np.asarray(r, dtype=float), device=self._ctx.device if self._ctx else None)
        r = nat.dev_f64(r, None, "r")
        return self.apply_into(r, torch.empty_like(r))

    def info(self):
        f, c, b = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        nat.check(nat.lib().acch_precond_info(self._handle, ctypes.byref(f), ctypes.byref(c), ctypes.byref(b)), "info")
        return {"factorizations": f.value, "classes": c.value, "factor_bytes": b.value}

    def __del__(self):
        if getattr(self, "_handle", None) is not None and nat._lib is not None:
            try:
                nat._lib.acch_precond_destroy(self._handle)
            except Exception:
                pass
            self._handle = None


# ---------------------------------------------------------------------------
# GMRES (linalg.py:403-506)
# ---------------------------------------------------------------------------

@dataclass
class GmresResult:
    x: torch.Tensor
    iterations: int
    converged: bool
    residual_norm: float


ORTHO = {"mgs": 0, "cgs2": 1, "dcgs2": 2}


def _generic_ctx(device):
    """A context for the grid-independent vector kernels (dot / axpby)."""
    from .physics import DEFAULT_PARAMS
    return nat.context_for(Grid((4, 4), (1.0, 1.0), BoundaryCondition.PERIODIC), DEFAULT_PARAMS, device)


def _gmres_generic(matvec, b, precond, rel_tol, abs_tol, restart, max_iterations, x0) -> GmresResult:
    """The reference's GMRES (linalg.py:411-506) for an arbitrary device
    matvec / preconditioner callable: the reference's operation order (MGS,
    second pass when ||w|| < ||w_0|| / 2, Givens, true-residual restarts),
    vectors on the device through the library's deterministic dot / axpby
    kernels, the (restart+1) x restart Hessenberg matrix on the host."""
    as_numpy = isinstance(b, np.ndarray) or np.isscalar(b)
    dev = b.device if isinstance(b, torch.Tensor) and b.is_cuda else torch.device("cuda", torch.cuda.current_device())
    bt = torch.as_tensor(np.asarray(b, dtype=float) if as_numpy else b, dtype=torch.float64, device=dev).reshape(-1)
    bt = bt.contiguous()
    n = bt.numel()
    ctx = _generic_ctx(dev)
    L = nat.lib()

    def to_dev(y):
        t = torch.as_tensor(np.asarray(y, dtype=float) if isinstance(y, np.ndarray) else y, dtype=torch.float64,
                            device=dev).reshape(-1)
        return t.contiguous()

    def dot(a, c):
        out = ctypes.c_double()
        nat.check(L.acch_dot(ctx.bind(), nat.ptr(a), nat.ptr(c), n, ctypes.byref(out)), "dot")
        return out.value

    def axpby(a, xv, bb, yv):      # yv <- a xv + bb yv
        nat.check(L.acch_axpby(ctx.bind(), float(a), nat.ptr(xv), float(bb), nat.ptr(yv), n), "axpby")

    if precond is None:
        apply_m = lambda v: v   # noqa: E731
    elif hasattr(precond, "apply"):
        apply_m = precond.apply
    else:
        apply_m = precond
    tol = max(rel_tol * math.sqrt(dot(bt, bt)), abs_tol)
    if x0 is None:
        x = torch.zeros_like(bt)
        r = bt.clone()
    else:
        x = to_dev(x0).clone()
        r = bt.clone()
        axpby(-1.0, to_dev(matvec(x)).clone(), 1.0, r)
    total = 0
    res_norm = math.sqrt(dot(r, r))
    while True:
        if res_norm <= tol:
            break
        if total >= max_iterations:
            break
        V = torch.zeros((restart + 1, n), dtype=torch.float64, device=dev)
        H = np.zeros((restart + 1, restart))
        cs = np.zeros(restart)
        sn = np.zeros(restart)
        g = np.zeros(restart + 1)
        axpby(1.0 / res_norm, r, 0.0, V[0])
        g[0] = res_norm
        j = 0
        breakdown = False
        while j < restart and total < max_iterations:
            # copy: matvec / preconditioner may hand back their input
            w = to_dev(matvec(to_dev(apply_m(V[j])))).clone()
            norm_before = math.sqrt(dot(w, w))
            for i in range(j + 1):
                H[i, j] = dot(V[i], w)
                axpby(-H[i, j], V[i], 1.0, w)
            norm_after = math.sqrt(dot(w, w))
            if norm_after < 0.5 * norm_before:
                for i in range(j + 1):
                    corr = dot(V[i], w)
                    H[i, j] += corr
                    axpby(-corr, V[i], 1.0, w)
                norm_after = math.sqrt(dot(w, w))
            H[j + 1, j] = norm_after
            total += 1
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            denom = math.hypot(H[j, j], H[j + 1, j])
            if denom == 0.0:
                breakdown = True
                break
            cs[j] = H[j, j] / denom
            sn[j] = H[j + 1, j] / denom
            H[j, j] = denom
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            j += 1
            if norm_after == 0.0:
                breakdown = True
                break
            axpby(1.0 / norm_after, w, 0.0, V[j])
            if abs(g[j]) <= tol:
                break
        if j > 0:
            y = np.zeros(j)
            for i in range(j - 1, -1, -1):
                y[i] = (g[i] - H[i, i + 1:j] @ y[i + 1:j]) / H[i, i]
            comb = torch.zeros_like(bt)
            for i in range(j):
                axpby(y[i], V[i], 1.0, comb)
            axpby(1.0, to_dev(apply_m(comb)).clone(), 1.0, x)
        r = bt.clone()
        axpby(-1.0, to_dev(matvec(x)).clone(), 1.0, r)
        res_norm = math.sqrt(dot(r, r))
        if breakdown and res_norm > tol:
            xo = x.cpu().numpy() if as_numpy else x
            return GmresResult(xo, total, False, res_norm)
    xo = x.cpu().numpy() if as_numpy else x
    return GmresResult(xo, total, res_norm <= tol, res_norm)


def gmres(matvec, b, precond=None, rel_tol: float = 1e-8, abs_tol: float = 1e-14, restart: int = 30,
          max_iterations: int = 500, x0=None, ortho: str = "dcgs2") -> GmresResult:
    """Restarted right-preconditioned GMRES (linalg.py:411-506).

    With a JacobianOperator (or its bound ``matvec``) and ``precond`` None or
    a SchwarzPreconditioner, the whole solve runs in libacch_b200 (device
    basis, device Hessenberg / Givens, no host round trip per Arnoldi step).
    ``ortho='mgs'`` reproduces the reference's modified Gram-Schmidt operation
    order; ``'cgs2'`` is classical Gram-Schmidt with the reference's
    conditional second pass, fused into two sweeps over the basis;
    ``'dcgs2'`` lags the second pass by one Arnoldi step (always taken) so
    that one multi-dot and one fused update sweep the basis per step
    (default).  Any other matvec (a callable on device vectors, e.g. a dense
    torch matrix) or preconditioner callable runs the reference's MGS
    algorithm through the library's vector kernels.  Stopping and restarts
    follow the reference: the recomputed true residual decides convergence;
    ``x0`` (default 0) is the initial guess."""
    from .scheme import JacobianOperator
    op = matvec
    if not isinstance(op, JacobianOperator):
        op = getattr(matvec, "__self__", None)
    native = isinstance(op, JacobianOperator) and (precond is None or isinstance(precond, SchwarzPreconditioner))
    if native and isinstance(b, torch.Tensor) and restart <= 32:
        if precond is not None and precond.handle is None:
            raise RuntimeError("preconditioner has no factorization; call update() first")
        b = nat.dev_f64(b, 2 * op.n_store, "b")
        if x0 is None:
            x = torch.empty_like(b)
        else:
            x = nat.dev_f64(torch.as_tensor(x0, dtype=torch.float64, device=b.device).reshape(-1).clone(),
                            2 * op.n_store, "x0")
        its, conv, rn = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_double()
        nat.check(nat.lib().acch_gmres_x0(op.ctx.bind(), nat.ptr(op.coef), op.dt,
                                          precond.handle if precond is not None else None, nat.ptr(b), nat.ptr(x),
                                          int(x0 is not None), float(rel_tol), float(abs_tol), int(restart),
                                          int(max_iterations), ORTHO[ortho], ctypes.byref(its), ctypes.byref(conv),
                                          ctypes.byref(rn)), "gmres")
        return GmresResult(x, int(its.value), bool(conv.value), float(rn.value))
    if restart < 1:
        raise ValueError("restart must be >= 1")
    return _gmres_generic(matvec, b, precond, rel_tol, abs_tol, restart, max_iterations, x0)


__all__ = ["Decomposition", "partition", "SchwarzVariant", "SubdomainSolverSpec", "SchwarzPreconditioner",
           "GmresResult", "gmres", "BoundaryCondition"]
