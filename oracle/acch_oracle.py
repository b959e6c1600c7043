"""CPU oracle for the AC/CH Newton-Krylov-Schwarz time step.

TEST INFRASTRUCTURE ONLY.  This module is the checker, never the product:
only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import it.  The product path
(``paper_2007_04560_b200``) never imports it and has no CPU fallback.

It restates, in plain numpy (plus the small C kernels in ``ilu_oracle.c`` for
the incomplete-LU numerics), the algorithm of the reference package ``acch``
under ``/root/reference/pkg/src/acch``.  Every function cites the reference
``file:line`` it follows.  The reference itself is pure Python; it is imported
only by ``tests/golden/make_golden.py`` (in the build container) to produce
the golden vectors under ``tests/golden/`` that pin this oracle
(``tests/test_oracle_golden.py``).  Parity status: PINNED against those
fixtures (residual, Jacobian, partition, ILU/LU Schwarz applies, GMRES,
Newton reports and whole ``simulate`` histories).

Vector layout follows the reference: solver vectors interleave (u, v) per
cell, cells x-fastest (scheme.py:58-80).  Arrays are stored with the axis
order reversed, (ny, nx) or (nz, ny, nx) (grid.py:80-86).
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field

import numpy as np
from scipy import sparse
from scipy.sparse.linalg import splu

ADMISSIBILITY_MARGIN = 1e-12          # physics.py:26
CHORD_BRANCH_FACTOR = 0.4             # physics.py:28-32


class OracleError(Exception):
    pass


class OInadmissible(OracleError):
    """Mirror of acch.exceptions.InadmissibleStateError (physics.py:116-121)."""


class OZeroPivot(OracleError):
    """Mirror of acch.exceptions.ZeroPivotError (exceptions.py:22-37)."""

    def __init__(self, cell, component):
        self.cell, self.component = int(cell), int(component)
        super().__init__(f"zero pivot at cell {cell}, component {component}")


class OStall(OracleError):
    """Mirror of acch.exceptions.SolverStallError (timestep.py:64-86)."""


# ---------------------------------------------------------------------------
# mesh and stencils  (grid.py:29-308)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Mesh:
    counts: tuple          # (nx, ny[, nz])
    lengths: tuple
    periodic: bool

    @property
    def dim(self):
        return len(self.counts)

    @property
    def shape(self):       # reversed-axis storage, x fastest (grid.py:80-86)
        return tuple(reversed(self.counts))

    @property
    def h(self):
        return tuple(L / n for L, n in zip(self.lengths, self.counts))

    @property
    def n_cells(self):
        return int(np.prod(self.counts))

    @property
    def cell_volume(self):
        return float(np.prod(self.h))

    def np_axis(self, axis):
        return self.dim - 1 - axis


def _ghosted(mesh: Mesh, a):
    """One ghost layer: wrap (periodic) or copy of the adjacent cell (Neumann).

    Same values as grid.py:177-194 (axis-sequential fill gives consistent
    corners, which np.pad's wrap/edge modes also produce)."""
    return np.pad(a, 1, mode="wrap" if mesh.periodic else "edge")


def _interior_but(ndim, na, sl):
    idx = [slice(1, -1)] * ndim
    idx[na] = sl
    return tuple(idx)


def laplacian(mesh: Mesh, a):
    """5/7-point Laplacian, axes summed in x, y, z order (grid.py:263-271)."""
    g = _ghosted(mesh, a)
    out = np.zeros(mesh.shape)
    nd = a.ndim
    for ax in range(mesh.dim):
        na = mesh.np_axis(ax)
        d = mesh.h[ax]
        plus = g[_interior_but(nd, na, slice(2, None))]
        minus = g[_interior_but(nd, na, slice(0, -2))]
        out += (plus - 2.0 * a + minus) / (d * d)
    return out


def face_means(mesh: Mesh, c):
    """Per-axis face averages of a cell field, N+1 faces along the axis
    (grid.py:235-246)."""
    g = _ghosted(mesh, c)
    out = []
    for ax in range(mesh.dim):
        na = mesh.np_axis(ax)
        line = g[_interior_but(c.ndim, na, slice(None))]
        n = line.shape[na]
        lo = [slice(None)] * c.ndim
        hi = [slice(None)] * c.ndim
        lo[na] = slice(0, n - 1)
        hi[na] = slice(1, n)
        out.append(0.5 * (line[tuple(lo)] + line[tuple(hi)]))
    return out


def div_c_grad(mesh: Mesh, cfaces, gcell):
    """Conservative flux difference div(c grad g) (grid.py:274-298)."""
    g = _ghosted(mesh, gcell)
    out = np.zeros(mesh.shape)
    for ax in range(mesh.dim):
        na = mesh.np_axis(ax)
        d = mesh.h[ax]
        line = g[_interior_but(gcell.ndim, na, slice(None))]
        n = line.shape[na]
        lo = [slice(None)] * gcell.ndim
        hi = [slice(None)] * gcell.ndim
        lo[na] = slice(0, n - 1)
        hi[na] = slice(1, n)
        flux = cfaces[ax] * (line[tuple(hi)] - line[tuple(lo)])
        flo = [slice(None)] * gcell.ndim
        fhi = [slice(None)] * gcell.ndim
        flo[na] = slice(0, n - 2)
        fhi[na] = slice(1, n - 1)
        out += (flux[tuple(fhi)] - flux[tuple(flo)]) / (d * d)
    return out


def grad_sq_avg(mesh: Mesh, a):
    """Per axis ((D+ a)^2 + (D- a)^2)/2, summed (grid.py:249-260)."""
    g = _ghosted(mesh, a)
    out = np.zeros(mesh.shape)
    for ax in range(mesh.dim):
        na = mesh.np_axis(ax)
        d = mesh.h[ax]
        fwd = (g[_interior_but(a.ndim, na, slice(2, None))] - a) / d
        bwd = (a - g[_interior_but(a.ndim, na, slice(0, -2))]) / d
        out += 0.5 * (fwd * fwd + bwd * bwd)
    return out


# ---------------------------------------------------------------------------
# constitutive functions  (physics.py:35-351)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Coeffs:
    alpha: float = 4.0
    beta: float = 2.0
    gamma: float = 0.005
    theta: float = 0.1
    rho: float = 0.001
    series_order: int = 10


def admissibility_gap(u, v):
    """min of u, 1-u, u±v, 1-(u±v), 1/2±v; NaN -> -inf (physics.py:89-109)."""
    p, q = u + v, u - v
    cands = [u.min(), (1.0 - u).min(), p.min(), (1.0 - p).min(), q.min(),
             (1.0 - q).min(), (0.5 - v).min(), (0.5 + v).min()]
    gap = float(min(cands))
    return -math.inf if math.isnan(gap) else gap


def require_admissible(u, v, margin=ADMISSIBILITY_MARGIN):
    gap = admissibility_gap(u, v)
    if not gap >= margin:
        raise OInadmissible(f"gap {gap:.3e} < {margin:.1e}")


def mobility(u, v):
    """c(u, v) = u (1 - u) (1/4 - v^2)  (physics.py:124-130)."""
    return u * (1.0 - u) * (0.25 - v * v)


def mobility_partials(u, v):
    """(dc/du, dc/dv)  (physics.py:133-135)."""
    return (1.0 - 2.0 * u) * (0.25 - v * v), -2.0 * v * u * (1.0 - u)


def entropy(z):
    """Phi(z) = z ln z + (1-z) ln(1-z)  (physics.py:160-166)."""
    return z * np.log(z) + (1.0 - z) * np.log1p(-z)


def entropy_prime(z):
    return np.log(z) - np.log1p(-z)


def _series_coefficients(order):
    """1/((2s+1) 2s) and 1/(2s+1), s = 1..order  (physics.py:178-182)."""
    s = np.arange(1, order + 1, dtype=float)
    return 1.0 / ((2.0 * s + 1.0) * 2.0 * s), 1.0 / (2.0 * s + 1.0)


def _horner_no_const(coeffs, t):
    """sum_s coeffs[s-1] t^s, acc = (acc + c_s) t from s = S down to 1
    (physics.py:185-190)."""
    acc = np.zeros_like(t)
    for c in coeffs[::-1]:
        acc = (acc + c) * t
    return acc


def chord(a, b, order=10, want_deriv=False, force_exact=False):
    """Divided difference (Phi(a)-Phi(b))/(a-b) with exact / series / direct
    branches (physics.py:213-262) and optionally d/da (physics.py:265-310)."""
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    a, b = np.broadcast_arrays(a, b)
    zeta = 0.5 * (a + b)
    sigma = 0.5 * (a - b)
    exact = sigma == 0.0
    if force_exact:
        near = np.zeros_like(exact)
    else:
        near = (np.abs(sigma) <= CHORD_BRANCH_FACTOR * np.minimum(zeta, 1.0 - zeta)) & ~exact
    far = ~(exact | near)
    val = np.empty(zeta.shape)
    der = np.empty(zeta.shape)
    c1, c2 = _series_coefficients(int(order))
    if exact.any():
        z = zeta[exact]
        val[exact] = np.log(z) - np.log1p(-z)
        der[exact] = 0.5 * (1.0 / z + 1.0 / (1.0 - z))
    if near.any():
        z, s = zeta[near], sigma[near]
        w = 1.0 - z
        rz, rw = s / z, s / w
        tz, tw = rz * rz, rw * rw
        val[near] = np.log(z) - np.log1p(-z) - _horner_no_const(c1, tz) + _horner_no_const(c1, tw)
        if want_deriv:
            qz = _horner_no_const(c2, tz)
            qw = _horner_no_const(c2, tw)
            der[near] = 0.5 * ((1.0 + qz) / z + (-qz / s) + (1.0 + qw) / w - (-qw / s))
    if far.any():
        af, bf = a[far], b[far]
        ch = (entropy(af) - entropy(bf)) / (af - bf)
        val[far] = ch
        der[far] = (entropy_prime(af) - ch) / (af - bf)
    if want_deriv:
        return val, der
    return val


def local_energy(co: Coeffs, u, v, gsu, gsv):
    """physics.py:313-322."""
    e1 = 0.5 * co.alpha * u * (1.0 - u) - 0.5 * co.beta * v * v
    e2 = co.theta * (entropy(u + v) + entropy(u - v))
    return e1 + e2 + 0.5 * co.gamma * (gsu + gsv)


def total_energy(mesh: Mesh, co: Coeffs, u, v):
    """<e> over all cells (physics.py:325-331)."""
    e = local_energy(co, u, v, grad_sq_avg(mesh, u), grad_sq_avg(mesh, v))
    return float(np.sum(e)) * mesh.cell_volume


# ---------------------------------------------------------------------------
# step residual and Jacobian  (scheme.py)
# ---------------------------------------------------------------------------

def pack(u, v):
    """Interleaved (u, v) per cell (scheme.py:62-66)."""
    out = np.empty(2 * u.size)
    out[0::2] = u.ravel()
    out[1::2] = v.ravel()
    return out


def unpack(mesh: Mesh, x):
    return x[0::2].reshape(mesh.shape), x[1::2].reshape(mesh.shape)


@dataclass
class Step:
    """Frozen data of one implicit step (scheme.py:195-246)."""

    mesh: Mesh
    co: Coeffs
    uo: np.ndarray
    vo: np.ndarray
    dt: float
    c_old: np.ndarray = field(init=False)
    lap_uo: np.ndarray = field(init=False)
    lap_vo: np.ndarray = field(init=False)

    def __post_init__(self):
        if not self.dt > 0.0:
            raise ValueError("time step must be positive")
        require_admissible(self.uo, self.vo)
        self.c_old = mobility(self.uo, self.vo)
        self.lap_uo = laplacian(self.mesh, self.uo)
        self.lap_vo = laplacian(self.mesh, self.vo)

    def dvd(self, un, vn, force_exact=False):
        """G_u, G_v of scheme.py:270-287."""
        co = self.co
        phi = chord(un + vn, self.uo + self.vo, co.series_order, force_exact=force_exact)
        psi = chord(un - vn, self.uo - self.vo, co.series_order, force_exact=force_exact)
        gu = (-0.5 * co.alpha * (un + self.uo - 1.0) + co.theta * (phi + psi)
              - 0.5 * co.gamma * (laplacian(self.mesh, un) + self.lap_uo))
        gv = (-0.5 * co.beta * (vn + self.vo) + co.theta * (phi - psi)
              - 0.5 * co.gamma * (laplacian(self.mesh, vn) + self.lap_vo))
        return gu, gv

    def residual_fields(self, un, vn):
        """F_u, F_v  (scheme.py:323-349); trapezoidal mobility as in
        scheme.py:223-232."""
        require_admissible(un, vn)
        gu, gv = self.dvd(un, vn)
        fo = face_means(self.mesh, self.c_old)
        fn = face_means(self.mesh, mobility(un, vn))
        mean_faces = [0.5 * (a + b) for a, b in zip(fo, fn)]
        cbar = 0.5 * (self.c_old + mobility(un, vn))
        fu = (un - self.uo) / self.dt + (-div_c_grad(self.mesh, mean_faces, gu))
        fv = (vn - self.vo) / self.dt + (cbar / self.co.rho) * gv
        return fu, fv

    def residual(self, x):
        un, vn = unpack(self.mesh, x)
        return pack(*self.residual_fields(un, vn))

    # -- Jacobian ------------------------------------------------------------

    def jacobian(self, x):
        return JacobianOracle(self, *unpack(self.mesh, x))


class JacobianOracle:
    """Matrix-free analytic Jacobian of the step residual.

    Equals scheme.py:427-484 (assembled block form) term by term: the u rows
    are w/dt - div(cbar grad dG_u) - div(dc grad G_u) with dG_u the
    linearised DVD and dc = 1/2 (c_u w_u + c_v w_v) the linearised
    trapezoidal mobility (scheme.py:357-424); the v rows are local plus a
    Laplacian (scheme.py:478-482)."""

    def __init__(self, step: Step, un, vn):
        require_admissible(un, vn)
        co = step.co
        self.step = step
        self.mesh = step.mesh
        _, dp = chord(un + vn, step.uo + step.vo, co.series_order, want_deriv=True)
        _, dq = chord(un - vn, step.uo - step.vo, co.series_order, want_deriv=True)
        self.S = co.theta * (dp + dq)
        self.D = co.theta * (dp - dq)
        self.cbar = 0.5 * (step.c_old + mobility(un, vn))
        self.cu, self.cv = mobility_partials(un, vn)
        self.gu, self.gv = step.dvd(un, vn)
        self.cbar_faces = face_means(self.mesh, self.cbar)

    def matvec_fields(self, wu, wv):
        co, st, m = self.step.co, self.step, self.mesh
        dgu = (-0.5 * co.alpha + self.S) * wu + self.D * wv - 0.5 * co.gamma * laplacian(m, wu)
        eta = 0.5 * (self.cu * wu + self.cv * wv)
        yu = wu / st.dt - div_c_grad(m, self.cbar_faces, dgu) - div_c_grad(m, face_means(m, eta), self.gu)
        yv = (wv / st.dt
              + (self.cbar / co.rho) * (self.D * wu + (-0.5 * co.beta + self.S) * wv
                                        - 0.5 * co.gamma * laplacian(m, wv))
              + (self.gv / co.rho) * eta)
        return yu, yv

    def matvec(self, w):
        return pack(*self.matvec_fields(*unpack(self.mesh, w)))

    def assemble(self):
        """Block CSR (indptr, indices, blocks[nnzb,2,2]) on the radius-2
        skeleton I + D + D^2 (scheme.py:166-188), by structured probing."""
        return probe_blocks(self.mesh, self.matvec)

    def assemble_fast(self):
        """The same block CSR, assembled directly from the per-cell
        coefficients (vectorised over cells, one stencil offset at a time);
        tests pin it against ``assemble`` (probing of the matvec).  Used by
        the CPU baseline, where probing would dominate the timing."""
        m, co, st = self.mesh, self.step.co, self.step
        d = m.dim
        ih2 = [1.0 / (hh * hh) for hh in m.h]
        hg = 0.5 * co.gamma
        offs = [o for o in _stencil_offsets(d)]
        oid = {o: i for i, o in enumerate(offs)}
        units = [tuple((s if b == a else 0) for b in range(d)) for a in range(d) for s in (1, -1)]
        zero = tuple(0 for _ in range(d))

        def shift(f, o):
            g = f
            for a in range(d):
                if o[a]:
                    g = np.roll(g, -o[a], axis=m.np_axis(a))
            return g

        coords = np.indices(m.shape)

        def valid(o):
            if m.periodic:
                return np.ones(m.shape, dtype=bool)
            ok = np.ones(m.shape, dtype=bool)
            for a in range(d):
                c = coords[m.np_axis(a)] + o[a]
                ok &= (c >= 0) & (c < m.counts[a])
            return ok

        vmask = {u: valid(u).astype(float) for u in units}
        L = sum(vmask[u] * ih2[[a for a in range(d) if u[a]][0]] for u in units)
        blk = {o: np.zeros(m.shape + (2, 2)) for o in offs}
        cb, gu = self.cbar, self.gu
        ktot = np.zeros(m.shape)
        eta0 = np.zeros(m.shape)
        terms = []
        for u in units:
            a = [b for b in range(d) if u[b]][0]
            K = 0.5 * (cb + shift(cb, u)) * ih2[a] * vmask[u]
            et = -0.5 * (shift(gu, u) - gu) * ih2[a] * vmask[u]
            ktot += K
            eta0 += et
            terms.append((u, -K, et))
        terms.insert(0, (zero, ktot, eta0))
        for mo, wdg, weta in terms:
            A = -0.5 * co.alpha + shift(self.S, mo) + hg * shift(L, mo)
            b = blk[mo]
            b[..., 0, 0] += wdg * A + weta * 0.5 * shift(self.cu, mo)
            b[..., 0, 1] += wdg * shift(self.D, mo) + weta * 0.5 * shift(self.cv, mo)
            for u2 in units:
                a2 = [q for q in range(d) if u2[q]][0]
                tgt = tuple(x + y for x, y in zip(mo, u2))
                blk[tgt][..., 0, 0] += -wdg * hg * ih2[a2] * shift(vmask[u2], mo)
        blk[zero][..., 0, 0] += 1.0 / st.dt
        cr = cb / co.rho
        blk[zero][..., 1, 0] += cr * self.D + self.gv * self.cu / (2.0 * co.rho)
        blk[zero][..., 1, 1] += (1.0 / st.dt + cr * (-0.5 * co.beta + self.S) + hg * cr * L
                                 + self.gv * self.cv / (2.0 * co.rho))
        for u in units:
            a = [b for b in range(d) if u[b]][0]
            blk[u][..., 1, 1] += -hg * cr * ih2[a] * vmask[u]
        n = m.n_cells
        ids = np.arange(n).reshape(m.shape)
        rows, cols, vals = [], [], []
        for o in offs:
            ok = valid(o).ravel()
            rows.append(ids.ravel()[ok])
            cols.append(shift(ids, o).ravel()[ok])
            vals.append(blk[o].reshape(n, 2, 2)[ok])
        rows = np.concatenate(rows)
        cols = np.concatenate(cols)
        vals = np.concatenate(vals)
        keys = rows * n + cols
        uk, inv = np.unique(keys, return_inverse=True)
        out = np.zeros((len(uk), 2, 2))
        np.add.at(out, inv, vals)
        r = uk // n
        indptr = np.zeros(n + 1, dtype=np.int64)
        np.add.at(indptr, r + 1, 1)
        return np.cumsum(indptr), (uk % n).astype(np.int64), out


def _stencil_offsets(dim):
    """Offsets with |dx|+|dy|+|dz| <= 2 (the radius-2 skeleton)."""
    rng = range(-2, 3)
    if dim == 2:
        return [(x, y) for y in rng for x in rng if abs(x) + abs(y) <= 2]
    return [(x, y, z) for z in rng for y in rng for x in rng if abs(x) + abs(y) + abs(z) <= 2]


# ---------------------------------------------------------------------------
# skeleton and probing assembly
# ---------------------------------------------------------------------------

def neighbor_ids(mesh: Mesh):
    """For every cell, the flat ids of its +/- neighbours per axis; -1 where
    a Neumann wall cuts the link (divgrad_csr's dropped entries,
    scheme.py:87-146)."""
    ids = np.arange(mesh.n_cells, dtype=np.int64).reshape(mesh.shape)
    out = []
    for ax in range(mesh.dim):
        na = mesh.np_axis(ax)
        for s in (+1, -1):
            nb = np.roll(ids, -s, axis=na)
            if not mesh.periodic:
                edge = [slice(None)] * mesh.dim
                edge[na] = -1 if s > 0 else 0
                nb = nb.copy()
                nb[tuple(edge)] = -1
            out.append(nb.ravel())
    return out


def skeleton(mesh: Mesh):
    """Boolean CSR of cells within two valid neighbour links (incl. self)."""
    n = mesh.n_cells
    rows, cols = [], []
    for nb in neighbor_ids(mesh):
        ok = nb >= 0
        rows.append(np.nonzero(ok)[0])
        cols.append(nb[ok])
    adj = sparse.csr_matrix((np.ones(sum(len(r) for r in rows)),
                             (np.concatenate(rows), np.concatenate(cols))), shape=(n, n))
    adj.data[:] = 1.0
    eye = sparse.identity(n, format="csr")
    sk = (eye + adj + adj @ adj).tocsr()
    sk.sum_duplicates()
    sk.sort_indices()
    sk.data[:] = 1.0
    return sk


def _color_period(n, periodic):
    if not periodic:
        return min(5, n)
    for p in range(5, n + 1):
        if n % p == 0:
            return p
    return n


def probe_blocks(mesh: Mesh, matvec):
    """Extract the 2x2 blocks of a radius-2 operator on the skeleton by
    applying it to colour-class indicator vectors (distance-5 colouring)."""
    sk = skeleton(mesh)
    n = mesh.n_cells
    coords = np.indices(mesh.shape).reshape(mesh.dim, -1)   # reversed axes
    periods = [_color_period(mesh.counts[mesh.dim - 1 - k], mesh.periodic) for k in range(mesh.dim)]
    color = np.zeros(n, dtype=np.int64)
    for k in range(mesh.dim):
        color = color * periods[k] + coords[k] % periods[k]
    ncolor = int(np.prod(periods))
    rows = np.repeat(np.arange(n), np.diff(sk.indptr))
    colsk = sk.indices
    blocks = np.zeros((len(colsk), 2, 2))
    for c in range(ncolor):
        sel = color == c
        if not sel.any():
            continue
        for comp in range(2):
            e = np.zeros(2 * n)
            e[2 * np.nonzero(sel)[0] + comp] = 1.0
            y = matvec(e)
            hit = sel[colsk]
            blocks[hit, 0, comp] = y[2 * rows[hit]]
            blocks[hit, 1, comp] = y[2 * rows[hit] + 1]
    return sk.indptr.astype(np.int64), colsk.astype(np.int64), blocks


def blocks_to_csr(n_cells, indptr, indices, blocks):
    return sparse.bsr_matrix((blocks, indices, indptr), shape=(2 * n_cells, 2 * n_cells)).tocsr()


# ---------------------------------------------------------------------------
# domain decomposition  (linalg.py:122-210)
# ---------------------------------------------------------------------------

def _ordered_factorisations(n, k):
    if k == 1:
        return [(n,)]
    out = []
    for d in range(1, n + 1):
        if n % d == 0:
            out += [(d,) + rest for rest in _ordered_factorisations(n // d, k - 1)]
    return out


@dataclass
class Boxes:
    n_subdomains: int
    overlap: int
    factors: tuple
    owned: list
    extended: list
    owned_pos: list


def decompose(mesh: Mesh, nsub: int, overlap: int) -> Boxes:
    """Near-cubical boxes: minimise max/min edge over ordered factorisations
    (ties lexicographic), remainder cells to the first boxes, extension by
    ``overlap`` wrapped or clipped, ids sorted (linalg.py:161-210)."""
    if nsub < 1 or overlap < 0:
        raise OracleError("bad partition request")
    best = None
    for f in _ordered_factorisations(nsub, mesh.dim):
        if any(f[a] > mesh.counts[a] for a in range(mesh.dim)):
            continue
        edges = [mesh.counts[a] / f[a] for a in range(mesh.dim)]
        key = (max(edges) / min(edges), f)
        if best is None or key < best:
            best = key
    if best is None:
        raise OracleError("cannot partition")
    factors = best[1]
    ranges = []
    for a in range(mesh.dim):
        n, p = mesh.counts[a], factors[a]
        sizes = [n // p + (1 if i < n % p else 0) for i in range(p)]
        starts = np.concatenate([[0], np.cumsum(sizes)[:-1]])
        ranges.append([(int(s), int(s + z)) for s, z in zip(starts, sizes)])

    def flat(axes):
        # x-fastest flat ids; outer product in z, y, x order
        stride = 1
        grids = np.meshgrid(*reversed(axes), indexing="ij")
        ids = np.zeros(grids[0].shape, dtype=np.int64)
        for a in range(mesh.dim):
            ids += grids[mesh.dim - 1 - a] * stride
            stride *= mesh.counts[a]
        return ids.ravel()

    owned, ext, pos = [], [], []
    for box in np.ndindex(*reversed(factors)):
        idx = tuple(reversed(box))
        own_axes, ext_axes = [], []
        for a in range(mesh.dim):
            lo, hi = ranges[a][idx[a]]
            own_axes.append(np.arange(lo, hi, dtype=np.int64))
            if mesh.periodic:
                e = np.unique(np.arange(lo - overlap, hi + overlap) % mesh.counts[a])
            else:
                e = np.arange(max(lo - overlap, 0), min(hi + overlap, mesh.counts[a]))
            ext_axes.append(e.astype(np.int64))
        o = flat(own_axes)
        e = flat(ext_axes)
        owned.append(o)
        ext.append(e)
        pos.append(np.searchsorted(e, o))
    return Boxes(nsub, overlap, tuple(factors), owned, ext, pos)


# ---------------------------------------------------------------------------
# ILU(k) / LU subdomain solves  (linalg.py:249-317, _ilu.py)
# ---------------------------------------------------------------------------

_CLIB = None


def _clib():
    global _CLIB
    if _CLIB is None:
        here = os.path.dirname(os.path.abspath(__file__))
        path = os.path.join(here, "_build", "liboracle_ilu.so")
        if not os.path.exists(path):
            build_c()
        lib = ctypes.CDLL(path)
        p = ctypes.c_void_p
        lib.oracle_ilu_factor.argtypes = [ctypes.c_int64, p, p, p, p]
        lib.oracle_ilu_factor.restype = ctypes.c_int64
        lib.oracle_ilu_solve.argtypes = [ctypes.c_int64, p, p, p, p, p, p]
        lib.oracle_ilu_solve.restype = None
        _CLIB = lib
    return _CLIB


def build_c():
    """Compile ilu_oracle.c with gcc into oracle/_build/ (test infrastructure)."""
    import subprocess
    here = os.path.dirname(os.path.abspath(__file__))
    os.makedirs(os.path.join(here, "_build"), exist_ok=True)
    subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-o",
                           os.path.join(here, "_build", "liboracle_ilu.so"),
                           os.path.join(here, "ilu_oracle.c")])


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def fill_pattern(indptr, indices, level):
    """Level-of-fill ILU(level) pattern on the block graph: structural
    entries level 0, fill via k has level lev(i,k)+lev(k,j)+1, kept when
    <= level (_ilu.py:19-64).  Rows processed in order; each row's pending
    columns are scanned in increasing order."""
    n = len(indptr) - 1
    if level == 0:
        return np.asarray(indptr, np.int64).copy(), np.asarray(indices, np.int64).copy()
    import heapq
    rows_c, rows_l = [], []
    for i in range(n):
        lev = {int(c): 0 for c in indices[indptr[i]:indptr[i + 1]]}
        heap = sorted(c for c in lev if c < i)
        seen = set(heap)
        while heap:
            k = heapq.heappop(heap)
            lik = lev[k]
            if lik >= level:
                continue
            kc, kl = rows_c[k], rows_l[k]
            for j, lkj in zip(kc, kl):
                if j <= k:
                    continue
                cand = lik + lkj + 1
                if cand > level:
                    continue
                if j not in lev or cand < lev[j]:
                    lev[j] = cand
                    if j < i and j not in seen:
                        heapq.heappush(heap, j)
                        seen.add(j)
        cs = sorted(lev)
        rows_c.append(cs)
        rows_l.append([lev[c] for c in cs])
    ip = np.zeros(n + 1, dtype=np.int64)
    ip[1:] = np.cumsum([len(c) for c in rows_c])
    return ip, np.array([c for r in rows_c for c in r], dtype=np.int64)


def scalar_pattern(bindptr, bindices):
    """kron(P, ones(2,2)) pattern, sorted (_ilu.py:67-74)."""
    n = len(bindptr) - 1
    p = sparse.csr_matrix((np.ones(len(bindices)), bindices, bindptr), shape=(n, n))
    s = sparse.kron(p, np.ones((2, 2)), format="csr")
    s.sort_indices()
    return s.indptr.astype(np.int64), s.indices.astype(np.int64)


class IluOracle:
    """Scalar ILU(k) of one subdomain block matrix, numerics in C."""

    def __init__(self, bindptr, bindices, bvals, level, cells=None):
        fip, fix = fill_pattern(bindptr, bindices, level)
        self.ip, self.ix = scalar_pattern(fip, fix)
        n = len(self.ip) - 1
        self.diag = np.empty(n, dtype=np.int64)
        for i in range(n):
            lo, hi = self.ip[i], self.ip[i + 1]
            self.diag[i] = lo + np.searchsorted(self.ix[lo:hi], i)
        csr = blocks_to_csr(len(bindptr) - 1, bindptr, bindices, bvals)
        csr.sort_indices()
        rows = np.repeat(np.arange(n), np.diff(csr.indptr))
        keys_pat = np.repeat(np.arange(n), np.diff(self.ip)) * n + self.ix
        keys = rows * n + csr.indices
        self.data = np.zeros(len(self.ix))
        self.data[np.searchsorted(keys_pat, keys)] = csr.data
        bad = _clib().oracle_ilu_factor(n, _ptr(self.ip), _ptr(self.ix), _ptr(self.data), _ptr(self.diag))
        if bad >= 0:
            cell = int(bad) // 2
            if cells is not None:
                cell = int(cells[cell])
            raise OZeroPivot(cell, int(bad) % 2)

    def solve(self, b):
        b = np.ascontiguousarray(b, dtype=float)
        out = np.empty_like(b)
        _clib().oracle_ilu_solve(len(b), _ptr(self.ip), _ptr(self.ix), _ptr(self.data),
                                 _ptr(self.diag), _ptr(b), _ptr(out))
        return out


class LuOracle:
    def __init__(self, bindptr, bindices, bvals):
        csr = blocks_to_csr(len(bindptr) - 1, bindptr, bindices, bvals)
        self._lu = splu(csr.tocsc())

    def solve(self, b):
        return self._lu.solve(np.asarray(b, dtype=float))


def restrict_blocks(indptr, indices, blocks, cells):
    """Principal block submatrix on sorted cells (linalg.py:71-89)."""
    n = len(indptr) - 1
    lookup = np.full(n, -1, dtype=np.int64)
    lookup[cells] = np.arange(len(cells))
    ip = [0]
    ix, bv = [], []
    for c in cells:
        lo, hi = indptr[c], indptr[c + 1]
        loc = lookup[indices[lo:hi]]
        keep = loc >= 0
        ix.append(loc[keep])
        bv.append(blocks[lo:hi][keep])
        ip.append(ip[-1] + int(keep.sum()))
    return np.array(ip, dtype=np.int64), np.concatenate(ix), np.concatenate(bv)


def interleave(cells):
    d = np.empty(2 * len(cells), dtype=np.int64)
    d[0::2] = 2 * cells
    d[1::2] = 2 * cells + 1
    return d


class SchwarzOracle:
    """ASM / left-RAS / right-RAS with ILU(k) or LU subdomain solves
    (linalg.py:320-396)."""

    def __init__(self, boxes: Boxes, variant="ras-left", solver="ilu0", threads=1):
        self.threads = max(1, int(threads))
        self.boxes = boxes
        self.variant = variant
        self.solver = solver
        self.factors = None
        self.factorization_count = 0
        self.ext_dofs = [interleave(c) for c in boxes.extended]
        self.own_dofs = [interleave(c) for c in boxes.owned]
        self.own_pos = [interleave(p) for p in boxes.owned_pos]

    def invalidate(self):
        self.factors = None

    def update(self, blocks_csr, reuse=False):
        if reuse and self.factors is not None:
            return False
        ip, ix, bv = blocks_csr

        def one(cells):
            sip, six, sbv = restrict_blocks(ip, ix, bv, cells)
            if self.solver == "lu":
                return LuOracle(sip, six, sbv)
            return IluOracle(sip, six, sbv, int(self.solver[3:]), cells)
        self.factors = self._map(one, self.boxes.extended)
        self.factorization_count += 1
        return True

    def _map(self, fn, items):
        """Ordered map; threads only change wall time (parallel.py:12-40)."""
        if self.threads == 1:
            return [fn(i) for i in items]
        from concurrent.futures import ThreadPoolExecutor
        if not hasattr(self, "_pool"):
            self._pool = ThreadPoolExecutor(self.threads)
        return list(self._pool.map(fn, items))

    def apply(self, r):
        out = np.zeros_like(r)

        def solve(k):
            if self.variant == "ras-right":
                rk = np.zeros(len(self.ext_dofs[k]))
                rk[self.own_pos[k]] = r[self.own_dofs[k]]
            else:
                rk = r[self.ext_dofs[k]]
            return self.factors[k].solve(rk)
        parts = self._map(solve, range(len(self.factors)))
        for k, yk in enumerate(parts):
            if self.variant == "ras-left":
                out[self.own_dofs[k]] = yk[self.own_pos[k]]
            else:
                out[self.ext_dofs[k]] += yk
        return out


# ---------------------------------------------------------------------------
# GMRES  (linalg.py:403-506)
# ---------------------------------------------------------------------------

@dataclass
class GmresOut:
    x: np.ndarray
    iterations: int
    converged: bool
    residual_norm: float


def gmres(matvec, b, precond=None, rel_tol=1e-8, abs_tol=1e-14, restart=30, max_iterations=500):
    """Right-preconditioned restarted GMRES, modified Gram-Schmidt with one
    extra pass when the norm drops below half, Givens rotations, restart and
    stop decided on the recomputed true residual (linalg.py:411-506)."""
    M = precond if precond is not None else (lambda z: z)
    tol = max(rel_tol * float(np.linalg.norm(b)), abs_tol)
    x = np.zeros_like(b)
    r = b.copy()
    beta = float(np.linalg.norm(r))
    its = 0
    while True:
        if beta <= tol:
            return GmresOut(x, its, True, beta)
        if its >= max_iterations:
            return GmresOut(x, its, False, beta)
        V = [r / beta]
        H = np.zeros((restart + 1, restart))
        cs = np.zeros(restart)
        sn = np.zeros(restart)
        g = np.zeros(restart + 1)
        g[0] = beta
        j = 0
        broke = False
        while j < restart and its < max_iterations:
            w = np.array(matvec(M(V[j])), dtype=float)
            n0 = float(np.linalg.norm(w))
            for i in range(j + 1):
                H[i, j] = np.dot(V[i], w)
                w -= H[i, j] * V[i]
            n1 = float(np.linalg.norm(w))
            if n1 < 0.5 * n0:
                for i in range(j + 1):
                    c = np.dot(V[i], w)
                    H[i, j] += c
                    w -= c * V[i]
                n1 = float(np.linalg.norm(w))
            H[j + 1, j] = n1
            its += 1
            for i in range(j):
                hi, hk = H[i, j], H[i + 1, j]
                H[i, j] = cs[i] * hi + sn[i] * hk
                H[i + 1, j] = -sn[i] * hi + cs[i] * hk
            den = math.hypot(H[j, j], H[j + 1, j])
            if den == 0.0:
                broke = True
                break
            cs[j], sn[j] = H[j, j] / den, H[j + 1, j] / den
            H[j, j], H[j + 1, j] = den, 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            j += 1
            if n1 == 0.0:
                broke = True
                break
            V.append(w / n1)
            if abs(g[j]) <= tol:
                break
        if j > 0:
            y = np.zeros(j)
            for i in range(j - 1, -1, -1):
                y[i] = (g[i] - H[i, i + 1:j] @ y[i + 1:]) / H[i, i]
            x = x + M(np.array(V[:j]).T @ y)
        r = b - matvec(x)
        beta = float(np.linalg.norm(r))
        if broke and beta > tol:
            return GmresOut(x, its, False, beta)


# ---------------------------------------------------------------------------
# Newton  (newton.py:29-186)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class NewtonSettings:
    rel_tol: float = 1e-6
    abs_tol: float = 1e-13
    lin_rel_tol: float = 1e-8
    lin_abs_tol: float = 1e-14
    max_iterations: int = 50
    backtrack_factor: float = 0.5
    min_step: float = 1e-8
    sufficient_decrease: float = 1e-4
    gmres_restart: int = 30
    max_linear_iterations: int = 500
    reuse_factorization: bool = True
    refactor_on_entry: bool = True


@dataclass
class NewtonReport:
    converged: bool
    newton_iterations: int
    gmres_iterations: int
    residual_norm: float
    reason: str | None = None
    factorizations: int = 0


def feasible_cap(u, v, su, sv, margin=1e-12, fraction=0.9):
    """Largest lambda <= 1 (x0.9) keeping every affine bound (newton.py:75-99)."""
    cap = math.inf
    for val, slope, lo, hi in ((u, su, margin, 1.0 - margin),
                               (u + v, su + sv, margin, 1.0 - margin),
                               (u - v, su - sv, margin, 1.0 - margin),
                               (v, sv, -0.5 + margin, 0.5 - margin)):
        neg = slope < 0.0
        pos = slope > 0.0
        if neg.any():
            cap = min(cap, float(np.min((val[neg] - lo) / -slope[neg])))
        if pos.any():
            cap = min(cap, float(np.min((hi - val[pos]) / slope[pos])))
    if not math.isfinite(cap):
        return 1.0
    return min(1.0, fraction * cap)


def newton_solve(step: Step, x0, cfg: NewtonSettings, precond: SchwarzOracle, trace=None):
    """Inexact Newton with Armijo backtracking and admissibility rejection;
    divergence reported, never raised (newton.py:102-186)."""
    mesh = step.mesh
    require_admissible(*unpack(mesh, x0))
    x = x0.copy()
    f = step.residual(x)
    fn = float(np.linalg.norm(f))
    stop = max(cfg.rel_tol * fn, cfg.abs_tol)
    lin_total = 0
    facs = 0
    for m in range(cfg.max_iterations + 1):
        if trace is not None:
            trace.append(fn)
        if fn <= stop:
            return x, NewtonReport(True, m, lin_total, fn, None, facs)
        if m == cfg.max_iterations:
            break
        jac = step.jacobian(x)
        reuse = (not cfg.refactor_on_entry) if m == 0 else cfg.reuse_factorization
        if not (reuse and precond.factors is not None):
            precond.update(jac.assemble_fast(), reuse=False)
            facs += 1
        lin = gmres(jac.matvec, -f, precond.apply, cfg.lin_rel_tol, cfg.lin_abs_tol,
                    cfg.gmres_restart, cfg.max_linear_iterations)
        lin_total += lin.iterations
        if not lin.converged:
            return x, NewtonReport(False, m, lin_total, fn, "linear_solve_failed", facs)
        s = lin.x
        u, v = unpack(mesh, x)
        su, sv = unpack(mesh, s)
        lam = feasible_cap(u, v, su, sv)
        ok = False
        while lam >= cfg.min_step:
            cand = x + lam * s
            if admissibility_gap(*unpack(mesh, cand)) >= ADMISSIBILITY_MARGIN:
                ft = step.residual(cand)
                ftn = float(np.linalg.norm(ft))
                if ftn <= (1.0 - cfg.sufficient_decrease * lam) * fn:
                    ok = True
                    break
            lam *= cfg.backtrack_factor
        if not ok:
            return x, NewtonReport(False, m, lin_total, fn, "line_search_stalled", facs)
        x, f, fn = cand, ft, ftn
    return x, NewtonReport(False, cfg.max_iterations, lin_total, fn, "max_newton_iterations", facs)


# ---------------------------------------------------------------------------
# adaptive time step  (timestep.py:23-89)
# ---------------------------------------------------------------------------

class Controller:
    def __init__(self, dt_min, dt_max, eta, fixed_dt=None, max_retries_at_min=5):
        self.dt_min, self.dt_max, self.eta = float(dt_min), float(dt_max), float(eta)
        self.fixed_dt = fixed_dt
        self.max_retries_at_min = max_retries_at_min
        self.stalled = 0
        self.divergence_count = 0

    def initial_dt(self):
        return self.dt_min if self.fixed_dt is None else self.fixed_dt

    def predict_dt(self, x_now, x_prev, dt_prev):
        if self.fixed_dt is not None:
            return self.fixed_dt
        d = x_now - x_prev
        rate = float(np.sqrt(np.mean(d * d))) / dt_prev
        dt = max(self.dt_min, self.dt_max / np.sqrt(1.0 + self.eta * rate * rate))
        return min(dt, self.dt_max)

    def on_divergence(self, dt):
        if self.fixed_dt is not None:
            raise OStall("diverged in fixed-step mode")
        self.divergence_count += 1
        self.eta *= 2.0
        if dt <= self.dt_min * (1.0 + 1e-12):
            self.stalled += 1
            if self.stalled >= self.max_retries_at_min:
                raise OStall("diverged repeatedly at dt_min")
        else:
            self.stalled = 0
        return max(self.dt_min, dt / np.sqrt(2.0))

    def note_success(self):
        self.stalled = 0


# ---------------------------------------------------------------------------
# the time loop  (cli/drivers.py:26-184)
# ---------------------------------------------------------------------------

def initial_fields(mesh: Mesh, center, amplitude, seed):
    """u = c + U(-a, a) then v = U(-a, a) from one generator (drivers.py:26-46)."""
    rng = np.random.default_rng(seed)
    u = center + rng.uniform(-amplitude, amplitude, mesh.shape)
    v = rng.uniform(-amplitude, amplitude, mesh.shape)
    return u, v


@dataclass
class Row:
    step: int
    time: float
    dt: float
    energy: float
    mass_u: float
    max_abs_v: float
    newton: int
    gmres: int


def diagnostics(mesh, co, u, v):
    """energy, mass, max|v| of a history row (drivers.py:62-73)."""
    return (total_energy(mesh, co, u, v), float(np.sum(u)) * mesh.cell_volume,
            float(np.max(np.abs(v))))


def simulate(mesh, co, u0, v0, controller: Controller, horizon, nsub, overlap=1,
             variant="ras-left", solver="ilu0", newton_cfg=NewtonSettings(),
             max_steps=None, refreeze_every=1, threads=1):
    """Accepted-step loop with retries on divergence (drivers.py:76-184).
    Returns (status, rows, final x, events) where events lists
    (step, dt_tried, reason) for every divergence."""
    boxes = decompose(mesh, nsub, overlap)
    pre = SchwarzOracle(boxes, variant, solver, threads)
    u, v = u0.copy(), v0.copy()
    rows = [Row(0, 0.0, 0.0, *diagnostics(mesh, co, u, v), 0, 0)]
    events = []
    x_now = pack(u, v)
    x_prev = None
    dt_prev = None
    t = 0.0
    step = 0
    since = 0
    refreeze_every = max(1, refreeze_every)
    status = "completed"
    while t < horizon * (1.0 - 1e-12):
        if max_steps is not None and step >= max_steps:
            break
        step += 1
        dt = controller.initial_dt() if (step == 1 or x_prev is None) else \
            controller.predict_dt(x_now, x_prev, dt_prev)
        if since >= refreeze_every:
            pre.invalidate()
            since = 0
        nn = ng = 0
        try:
            while True:
                st = Step(mesh, co, *unpack(mesh, x_now), dt)
                x_new, rep = newton_solve(st, x_now, newton_cfg, pre)
                nn += rep.newton_iterations
                ng += rep.gmres_iterations
                if rep.converged:
                    break
                events.append((step, dt, rep.reason))
                dt = controller.on_divergence(dt)
                pre.invalidate()
                since = 0
        except OStall:
            status = "stalled"
            break
        since += 1
        controller.note_success()
        t += dt
        x_prev, x_now, dt_prev = x_now, x_new, dt
        rows.append(Row(step, t, dt, *diagnostics(mesh, co, *unpack(mesh, x_now)), nn, ng))
    return status, rows, x_now, events
