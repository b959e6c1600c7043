"""Drop-in API surface and the reference's property suite, on the GPU path.

* gmres with a generic device matvec / preconditioner callable and an
  initial guess x0 (linalg.py:411-439): the reference's dense oracles
  (pkg/tests/test_linalg.py:324-379) restated on torch matrices, plus x0
  through the native Krylov driver.
* admissibility_gap on (u, v) arrays (physics.py:89-109).
* DVD energy identity E(U') - E(U^n) = <G, U' - U^n> (test_scheme.py:88-104),
  Jacobian against central finite differences of the residual
  (test_scheme.py:258-297), and the operator's conservation, symmetry /
  semi-positivity and summation-by-parts identity (test_grid.py:322-382,
  test_scheme.py:148-160), all evaluated through the device kernels."""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2007_04560_b200.grid import BoundaryCondition, Grid  # noqa: E402
from paper_2007_04560_b200.linalg import (SchwarzPreconditioner, SchwarzVariant,  # noqa: E402
                                          SubdomainSolverSpec, gmres, partition)
from paper_2007_04560_b200.physics import (Params, State, admissibility_gap,  # noqa: E402
                                           diagnostics)
from paper_2007_04560_b200.scheme import (N_COEF, StepProblem, assemble_jacobian,  # noqa: E402
                                          prepare_jacobian_unchecked, residual_vector)

DEV = "cuda:0"
PARAMS = Params(4.0, 2.0, 0.005, 0.1, 0.001)
BOTH = [BoundaryCondition.PERIODIC, BoundaryCondition.NEUMANN]


def T(a):
    return torch.as_tensor(np.asarray(a, dtype=float), dtype=torch.float64, device=DEV)


def host(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


# --------------------------------------------------------------------------- generic GMRES

def test_gmres_identity_one_iteration(rng):
    b = rng.standard_normal(40)
    res = gmres(lambda x: x, b, rel_tol=1e-12)
    assert res.converged and res.iterations == 1
    np.testing.assert_allclose(res.x, b, rtol=1e-12, atol=1e-14)


def test_gmres_zero_rhs():
    res = gmres(lambda x: 2 * x, np.zeros(10))
    assert res.converged and res.iterations == 0
    assert np.all(res.x == 0.0)


def test_gmres_matches_dense_solve(rng):
    n = 50
    a = rng.standard_normal((n, n)) + 6.0 * np.eye(n)
    b = rng.standard_normal(n)
    at = T(a)
    res = gmres(lambda x: at @ x, b, rel_tol=1e-10, abs_tol=0.0, restart=60)
    assert res.converged
    np.testing.assert_allclose(res.x, np.linalg.solve(a, b), rtol=1e-6, atol=1e-10)
    assert np.linalg.norm(b - a @ res.x) <= 1e-10 * np.linalg.norm(b)


def test_gmres_ill_conditioned_true_residual(rng):
    d = np.logspace(0, 6, 64)
    b = rng.standard_normal(64)
    dt = T(d)
    res = gmres(lambda x: dt * x, b, rel_tol=1e-8, abs_tol=0.0, restart=70, max_iterations=500)
    assert res.converged
    true_res = np.linalg.norm(b - d * res.x)
    assert true_res <= 1e-8 * np.linalg.norm(b)
    assert res.residual_norm == pytest.approx(true_res, rel=1e-9)


def test_gmres_restart_path(rng):
    n = 80
    d = np.linspace(1.0, 300.0, n)
    a = (np.eye(n) + np.diag(0.4 * np.ones(n - 1), 1)) * d
    b = rng.standard_normal(n)
    at = T(a)
    res = gmres(lambda x: at @ x, b, rel_tol=1e-9, abs_tol=0.0, restart=15, max_iterations=400)
    assert res.converged and res.iterations > 15
    assert np.linalg.norm(b - a @ res.x) <= 1e-9 * np.linalg.norm(b)


def test_gmres_iteration_cap(rng):
    d = T(np.logspace(0, 8, 128))
    b = rng.standard_normal(128)
    res = gmres(lambda x: d * x, b, rel_tol=1e-12, abs_tol=0.0, restart=10, max_iterations=20)
    assert not res.converged and res.iterations == 20


def test_gmres_generic_preconditioner_callable_and_x0(rng):
    """A preconditioner given as a plain callable (Jacobi) and an x0: the
    answer is the dense solve, and starting from the solution takes 0
    iterations (linalg.py:437-442)."""
    n = 60
    a = rng.standard_normal((n, n)) + 8.0 * np.eye(n)
    b = rng.standard_normal(n)
    at, dinv = T(a), T(1.0 / np.diag(a))
    res = gmres(lambda x: at @ x, T(b), precond=lambda r: dinv * r, rel_tol=1e-11, abs_tol=0.0, restart=40)
    assert res.converged
    xs = np.linalg.solve(a, b)
    np.testing.assert_allclose(host(res.x), xs, rtol=1e-8, atol=1e-10)
    again = gmres(lambda x: at @ x, T(b), rel_tol=1e-8, abs_tol=0.0, x0=T(xs))
    assert again.converged and again.iterations == 0


def _jac_case(bc=BoundaryCondition.PERIODIC):
    g = Grid((16, 12), (1.0, 1.0), bc)
    rng = np.random.default_rng(5)
    u = 0.5 + rng.uniform(-0.1, 0.1, g.array_shape)
    v = rng.uniform(-0.1, 0.1, g.array_shape)
    old = State.from_interior(g, u, v, device=DEV)
    prob = StepProblem.create(g, PARAMS, old, 1e-3)
    new = State.from_interior(g, u + 1e-3 * rng.standard_normal(g.array_shape),
                              v + 1e-3 * rng.standard_normal(g.array_shape), device=DEV)
    J = assemble_jacobian(prob, new)
    pre = SchwarzPreconditioner(partition(g, 4, 1), SchwarzVariant.LEFT_RAS, SubdomainSolverSpec("ilu", 0))
    pre.update(J)
    return g, prob, new, J, pre, torch.tensor(rng.standard_normal(2 * g.n_cells), device=DEV)


@pytest.mark.parametrize("ortho", ["mgs", "cgs2", "dcgs2"])
def test_native_gmres_x0(ortho):
    """x0 through the library's driver: the solution from a good initial guess
    equals the cold-start one, in fewer iterations; a converged x0 takes 0."""
    g, prob, new, J, pre, b = _jac_case()
    cold = gmres(J, b, pre, 1e-10, 1e-14, 30, 500, ortho=ortho)
    assert cold.converged
    x0 = cold.x + 1e-4 * torch.randn_like(cold.x) * cold.x.abs().max()
    warm = gmres(J, b, pre, 1e-10, 1e-14, 30, 500, x0=x0, ortho=ortho)
    assert warm.converged and warm.iterations < cold.iterations
    assert torch.linalg.norm(warm.x - cold.x) <= 1e-8 * torch.linalg.norm(cold.x)
    # ||b - J x|| of the returned x is the reported residual norm
    r = b - J.matvec(warm.x)
    assert float(torch.linalg.norm(r)) == pytest.approx(warm.residual_norm, rel=1e-6)
    done = gmres(J, b, pre, 1e-10, 1e-14, 30, 500, x0=cold.x, ortho=ortho)
    assert done.converged and done.iterations == 0


def test_generic_and_native_gmres_agree():
    """The Jacobian handed over as an opaque callable (generic MGS path) and
    as a JacobianOperator (native driver) give the same solution."""
    g, prob, new, J, pre, b = _jac_case(BoundaryCondition.NEUMANN)
    nat = gmres(J, b, pre, 1e-10, 1e-14, 30, 500, ortho="mgs")
    gen = gmres(lambda w: J.matvec(w), b, lambda r: pre.apply(r), 1e-10, 1e-14, 30, 500)
    assert nat.converged and gen.converged
    assert abs(nat.iterations - gen.iterations) <= 1
    assert torch.linalg.norm(nat.x - gen.x) <= 1e-8 * torch.linalg.norm(nat.x)


# --------------------------------------------------------------------------- admissibility gap

def _gap_ref(u, v):
    p, q = u + v, u - v
    gap = min(np.min(u), np.min(1 - u), np.min(p), np.min(1 - p), np.min(q), np.min(1 - q), np.min(0.5 - v),
              np.min(0.5 + v))
    return -np.inf if np.isnan(gap) else float(gap)


def test_admissibility_gap_arrays(rng):
    u = 0.5 + rng.uniform(-0.2, 0.2, (7, 9))
    v = rng.uniform(-0.2, 0.2, (7, 9))
    assert admissibility_gap(u, v) == _gap_ref(u, v)
    assert admissibility_gap(T(u), T(v)) == _gap_ref(u, v)
    u2 = u.copy()
    u2[3, 4] = 1.2
    assert admissibility_gap(u2, v) == _gap_ref(u2, v) < 0
    u2[1, 1] = np.nan
    assert admissibility_gap(u2, v) == -np.inf
    assert admissibility_gap(0.5, 0.0) == 0.5   # scalars broadcast
    g = Grid((9, 7), (1.0, 1.0), BoundaryCondition.PERIODIC)
    s = State.from_interior(g, u, v, device=DEV)
    assert admissibility_gap(s) == _gap_ref(u, v)


# --------------------------------------------------------------------------- properties

def _coef_fields(prob, x):
    """(cbar, G_u, G_v) per cell from the Jacobian coefficient records."""
    n = prob.grid.n_store
    coef = torch.empty(N_COEF * n, dtype=torch.float64, device=DEV)
    prepare_jacobian_unchecked(prob, x, coef)
    c = host(coef)
    B = c[4 * n:6 * n].reshape(n, 2)
    return B[:, 0], B[:, 1], c[6 * n:7 * n]


@pytest.mark.parametrize("bc", BOTH)
@pytest.mark.parametrize("counts", [(16, 16), (32, 32), (8, 6, 5)])
def test_dvd_energy_identity(bc, counts):
    """E(U') - E(U^n) = <G_u, u' - u^n> + <G_v, v' - v^n> to 1e-11 relative
    (test_scheme.py:88-104).  The pairs are far apart (u^n near 0.25, u' near
    0.75), so every chord takes the direct-quotient branch, the exact chord
    the reference's identity test forces."""
    g = Grid(counts, tuple(1.0 for _ in counts), bc)
    rng = np.random.default_rng(31 + len(counts))
    for _ in range(3):
        uo = 0.25 + rng.uniform(-0.03, 0.03, g.array_shape)
        vo = rng.uniform(-0.02, 0.02, g.array_shape)
        un = 0.75 + rng.uniform(-0.03, 0.03, g.array_shape)
        vn = rng.uniform(-0.02, 0.02, g.array_shape)
        old = State.from_interior(g, uo, vo, device=DEV)
        new = State.from_interior(g, un, vn, device=DEV)
        prob = StepProblem.create(g, PARAMS, old, 1e-3)
        _, gu, gv = _coef_fields(prob, new.vector)
        rhs = g.cell_volume * (np.dot(gu, (un - uo).ravel()) + np.dot(gv, (vn - vo).ravel()))
        e_new = diagnostics(new, PARAMS)[0]
        e_old = diagnostics(old, PARAMS)[0]
        lhs = e_new - e_old
        assert abs(lhs - rhs) <= 1e-11 * max(abs(e_new), abs(e_old), abs(lhs))


def _fd_action(prob, base, w, eps):
    return (residual_vector(prob, base + eps * w) - residual_vector(prob, base - eps * w)) / (2 * eps)


@pytest.mark.parametrize("bc", BOTH)
@pytest.mark.parametrize("counts", [(12, 10), (6, 5, 4)])
def test_jacobian_matches_fd_near_pair(bc, counts):
    g = Grid(counts, tuple(1.0 for _ in counts), bc)
    rng = np.random.default_rng(7)
    uo = 0.5 + rng.uniform(-0.15, 0.15, g.array_shape)
    vo = rng.uniform(-0.15, 0.15, g.array_shape)
    old = State.from_interior(g, uo, vo, device=DEV)
    new = State.from_interior(g, uo + 0.02 * rng.standard_normal(g.array_shape),
                              vo + 0.02 * rng.standard_normal(g.array_shape), device=DEV)
    prob = StepProblem.create(g, PARAMS, old, 1e-3)
    J = assemble_jacobian(prob, new)
    base = new.vector.clone()
    for _ in range(3):
        w = torch.tensor(rng.standard_normal(base.numel()), device=DEV)
        w /= torch.sqrt(torch.mean(w * w))
        jw = J.matvec(w)
        err = torch.linalg.norm(jw - _fd_action(prob, base, w, 1e-6)) / torch.linalg.norm(jw)
        assert float(err) <= 1e-5


def test_jacobian_matches_fd_far_pair():
    g = Grid((10, 8), (1.0, 1.0), BoundaryCondition.PERIODIC)
    rng = np.random.default_rng(8)
    old = State.from_interior(g, 0.2 + rng.uniform(0.0, 0.05, g.array_shape),
                              rng.uniform(-0.02, 0.02, g.array_shape), device=DEV)
    new = State.from_interior(g, 0.75 + rng.uniform(0.0, 0.05, g.array_shape),
                              rng.uniform(-0.02, 0.02, g.array_shape), device=DEV)
    prob = StepProblem.create(g, PARAMS, old, 1e-2)
    J = assemble_jacobian(prob, new)
    w = torch.tensor(rng.standard_normal(2 * g.n_cells), device=DEV)
    w /= torch.sqrt(torch.mean(w * w))
    jw = J.matvec(w)
    err = torch.linalg.norm(jw - _fd_action(prob, new.vector.clone(), w, 1e-6)) / torch.linalg.norm(jw)
    assert float(err) <= 1e-5


def _operator_parts(prob, x):
    """A(U') = F(U') - (U' - U^n)/dt from two residual evaluations at
    different dt: A_u = -div(cbar grad G_u), A_v = (cbar/rho) G_v."""
    g = prob.grid
    F1 = host(residual_vector(prob, x)).reshape(-1, 2)
    prob2 = StepProblem.create(g, prob.params, prob.old, 2.0 * prob.dt)
    F2 = host(residual_vector(prob2, x)).reshape(-1, 2)
    # F1 - F2 = dU (1/dt - 1/(2 dt)) = dU / (2 dt)  ->  A = 2 F2 - F1
    return 2.0 * F2 - F1


def _face_sum(g, cbar, gu):
    """sum over faces of cbar_face (G_{i+1} - G_i)^2 / h^2 (SBP right side,
    test_grid.py:337-355 with phi = psi)."""
    shp = g.array_shape
    c = cbar.reshape(shp)
    G = gu.reshape(shp)
    tot = 0.0
    for axis in range(g.dim):
        na = g.dim - 1 - axis
        h2 = g.spacing[axis] ** 2
        if g.periodic:
            cf = 0.5 * (c + np.roll(c, -1, axis=na))
            dG = np.roll(G, -1, axis=na) - G
            tot += np.sum(cf * dG * dG) / h2
        else:
            lo = [slice(None)] * g.dim
            hi = [slice(None)] * g.dim
            lo[na] = slice(0, -1)
            hi[na] = slice(1, None)
            cf = 0.5 * (c[tuple(lo)] + c[tuple(hi)])
            dG = G[tuple(hi)] - G[tuple(lo)]
            tot += np.sum(cf * dG * dG) / h2
    return tot


@pytest.mark.parametrize("bc", BOTH)
@pytest.mark.parametrize("counts", [(12, 9), (5, 6, 4), (16, 16, 8)])
def test_operator_conservation_sbp_and_semipositivity(bc, counts):
    """On the device residual: sum(A_u) = 0 (mass conservation, the flux
    form telescopes), <G_u, A_u> = sum_faces cbar (dG_u)^2 / h^2 >= 0
    (summation by parts), <G_v, A_v> >= 0."""
    g = Grid(counts, tuple(1.0 for _ in counts), bc)
    rng = np.random.default_rng(11)
    uo = 0.5 + rng.uniform(-0.15, 0.15, g.array_shape)
    vo = rng.uniform(-0.15, 0.15, g.array_shape)
    old = State.from_interior(g, uo, vo, device=DEV)
    new = State.from_interior(g, uo + 0.02 * rng.standard_normal(g.array_shape),
                              vo + 0.02 * rng.standard_normal(g.array_shape), device=DEV)
    prob = StepProblem.create(g, PARAMS, old, 1e-3)
    A = _operator_parts(prob, new.vector)
    cbar, gu, gv = _coef_fields(prob, new.vector)
    scale = np.sum(np.abs(A[:, 0]))
    assert abs(np.sum(A[:, 0])) <= 1e-11 * scale
    lhs = float(np.dot(gu, A[:, 0]))
    rhs = _face_sum(g, cbar, gu)
    assert rhs >= 0.0
    assert abs(lhs - rhs) <= 1e-9 * (abs(lhs) + abs(rhs))
    assert float(np.dot(gv, A[:, 1])) >= 0.0
    np.testing.assert_allclose(A[:, 1], cbar / PARAMS.rho * gv, rtol=1e-9, atol=1e-9 * np.max(np.abs(A[:, 1])))


# --------------------------------------------------------------------------- output files

def test_simulate_writes_history_and_snapshots(tmp_path):
    """simulate(out_dir=...) writes the reference's history CSV (flushed per
    step) and VTK snapshots (requested times, every k steps, final), and the
    files read back to the run's values (cli/drivers.py:76-184, io.py)."""
    from paper_2007_04560_b200.drivers import (InitialSpec, OutputSpec, RunConfig, SolverSpec, TimeSpec,
                                               simulate)
    from paper_2007_04560_b200.io import read_history, read_vtk, state_from_vtk
    g = Grid((16, 16), (1.0, 1.0), BoundaryCondition.PERIODIC)
    cfg = RunConfig(g, PARAMS, InitialSpec("random_uniform", 0.5, 0.05, 1234),
                    TimeSpec(horizon=4e-4, mode="fixed", dt=1e-4), SolverSpec(subdomains=4),
                    OutputSpec(history="h.csv", snapshot_times=(2e-4,), snapshot_every=3))
    res = simulate(cfg, out_dir=str(tmp_path), device=DEV)
    rows = read_history(str(tmp_path / "h.csv"))
    assert [r.step for r in rows] == [r.step for r in res.history] == [0, 1, 2, 3, 4]
    for a, b in zip(rows, res.history):
        assert (a.time, a.dt, a.energy, a.mass_u, a.newton, a.gmres) == (b.time, b.dt, b.energy, b.mass_u, b.newton,
                                                                          b.gmres)
    assert (tmp_path / "snapshot_t0.0002.vtk").exists() and (tmp_path / "step_000003.vtk").exists()
    u, v = res.final_state.to_numpy()
    meta = read_vtk(str(tmp_path / "final.vtk"))
    np.testing.assert_array_equal(meta["arrays"]["u"], u.ravel())
    back = state_from_vtk(str(tmp_path / "final.vtk"), BoundaryCondition.PERIODIC, device=DEV)
    assert torch.equal(back.x, res.final_state.x)
