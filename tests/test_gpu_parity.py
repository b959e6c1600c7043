"""GPU parity: the sm_100a path (through the C ABI) against the reference's
golden vectors and the CPU oracle on the same seeded inputs.

Tolerances (north_star): fp64 residual relative error <= 1e-12; fields
after N steps <= 1e-8 relative L2; identical accepted dt sequence (1e-10
relative), identical Newton counts and retry events; mass conserved and the
discrete energy monotone."""

import numpy as np
import pytest
import torch

from conftest import golden

pytestmark = pytest.mark.gpu

from paper_2007_04560_b200.exceptions import InadmissibleStateError  # noqa: E402
from paper_2007_04560_b200.grid import BoundaryCondition, Grid  # noqa: E402
from paper_2007_04560_b200.linalg import (SchwarzPreconditioner, SchwarzVariant,  # noqa: E402
                                          SubdomainSolverSpec, gmres, partition)
from paper_2007_04560_b200.newton import NewtonConfig, newton_solve  # noqa: E402
from paper_2007_04560_b200.physics import (Params, State, entropy_chord,  # noqa: E402
                                           entropy_chord_with_deriv, is_admissible, diagnostics)
from paper_2007_04560_b200.scheme import (StepProblem, assemble_jacobian,  # noqa: E402
                                          residual_vector)

PARAMS = Params(4.0, 2.0, 0.005, 0.1, 0.001)
STENCIL = ["2d_neu", "2d_per", "2d_per4", "3d_neu", "3d_per", "2d_per_big", "3d_neu_big"]
DEV = "cuda:0"


def grid_of(z):
    counts = tuple(int(c) for c in z["counts"])
    bc = BoundaryCondition.PERIODIC if bool(z["periodic"]) else BoundaryCondition.NEUMANN
    return Grid(counts, tuple(1.0 for _ in counts), bc)


def st(grid, u, v):
    return State.from_interior(grid, u, v, device=DEV)


def host(t):
    return t.detach().cpu().numpy()


# --------------------------------------------------------------------------- physics

def test_chord_battery():
    z = golden("chord.npz")
    a = torch.tensor(z["a"], device=DEV)
    b = torch.tensor(z["b"], device=DEV)
    val, der = entropy_chord_with_deriv(a, b, 10)
    np.testing.assert_allclose(host(val), z["val"], rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(host(der), z["der"], rtol=1e-12, atol=1e-13)
    assert np.array_equal(host(entropy_chord(a, b)), host(val))


def test_chord_known_answers():
    assert entropy_chord(0.6, 0.4) == 0.0
    assert abs(entropy_chord(0.7, 0.5) - 0.41141439252525923) <= 1e-12


# --------------------------------------------------------------------------- scheme

@pytest.mark.parametrize("form", ["zm", "ring"])
@pytest.mark.parametrize("tag", STENCIL)
def test_residual_matches_reference(tag, form, monkeypatch):
    monkeypatch.setenv("ACCH_RESIDUAL", form)
    z = golden(f"stencil_{tag}.npz")
    g = grid_of(z)
    prob = StepProblem.create(g, PARAMS, st(g, z["uo"], z["vo"]), float(z["dt"]))
    F = host(residual_vector(prob, st(g, z["un"], z["vn"])))
    assert np.max(np.abs(F - z["F"])) <= 1e-12 * np.max(np.abs(z["F"]))
    F0 = host(residual_vector(prob, st(g, z["uo"], z["vo"])))
    assert np.max(np.abs(F0 - z["F0"])) <= 1e-12 * np.max(np.abs(z["F0"]))


@pytest.mark.parametrize("order", [6, 13])
@pytest.mark.parametrize("bc", [BoundaryCondition.PERIODIC, BoundaryCondition.NEUMANN])
def test_residual_runtime_series_order_matches_oracle(order, bc, monkeypatch):
    """A series order other than the compiled-in 10 (run-time Horner in the
    z-marching residual) against the oracle, near- and exact-branch states."""
    from oracle import acch_oracle as O
    monkeypatch.setenv("ACCH_RESIDUAL", "zm")
    rng = np.random.default_rng(21)
    counts = (12, 10, 9)
    g = Grid(counts, (1.0, 1.0, 1.0), bc)
    params = Params(4.0, 2.0, 0.005, 0.1, 0.001, order)
    uo, vo = 0.5 + rng.uniform(-0.05, 0.05, g.array_shape), rng.uniform(-0.05, 0.05, g.array_shape)
    un, vn = uo + rng.uniform(-0.02, 0.02, g.array_shape), vo + rng.uniform(-0.02, 0.02, g.array_shape)
    prob = StepProblem.create(g, params, st(g, uo, vo), 1e-3)
    m = O.Mesh(counts, (1.0, 1.0, 1.0), bc == BoundaryCondition.PERIODIC)
    so = O.Step(m, O.Coeffs(series_order=order), uo, vo, 1e-3)
    for a, b in ((un, vn), (uo, vo)):
        F = host(residual_vector(prob, st(g, a, b)))
        Fo = so.residual(O.pack(a, b))
        assert np.max(np.abs(F - Fo)) <= 1e-12 * np.max(np.abs(Fo))


@pytest.mark.parametrize("form", ["zm", "twopass", "fused"])
@pytest.mark.parametrize("tag", STENCIL)
def test_jacobian_matvec_matches_reference(tag, form, monkeypatch):
    monkeypatch.setenv("ACCH_MATVEC", form)
    z = golden(f"stencil_{tag}.npz")
    g = grid_of(z)
    prob = StepProblem.create(g, PARAMS, st(g, z["uo"], z["vo"]), float(z["dt"]))
    J = assemble_jacobian(prob, st(g, z["un"], z["vn"]))
    y = host(J.matvec(torch.tensor(z["w"], device=DEV)))
    assert np.max(np.abs(y - z["Jw"])) <= 1e-12 * np.max(np.abs(z["Jw"]))


@pytest.mark.parametrize("tag", ["2d_neu", "2d_per", "2d_per4", "3d_neu", "3d_per"])
def test_jacobian_blocks_match_reference_bsr(tag):
    from scipy import sparse
    z = golden(f"stencil_{tag}.npz")
    g = grid_of(z)
    prob = StepProblem.create(g, PARAMS, st(g, z["uo"], z["vo"]), float(z["dt"]))
    J = assemble_jacobian(prob, st(g, z["un"], z["vn"]))
    got = J.to_bsr().toarray()
    ref = sparse.bsr_matrix((z["J_blocks"], z["J_indices"], z["J_indptr"]),
                            shape=(2 * g.n_cells, 2 * g.n_cells)).toarray()
    assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref))
    # same structural skeleton (scheme.py:166-188)
    ip = J.to_bsr()
    ip.sort_indices()
    assert ip.indices.size == z["J_indices"].size


@pytest.mark.parametrize("tag", STENCIL)
def test_energy_and_gap_match_reference(tag):
    z = golden(f"stencil_{tag}.npz")
    g = grid_of(z)
    e, _, _ = diagnostics(st(g, z["un"], z["vn"]), PARAMS)
    assert abs(e - float(z["energy_new"])) <= 1e-13 * abs(float(z["energy_new"]))
    from paper_2007_04560_b200.physics import state_gap
    assert state_gap(st(g, z["un"], z["vn"])) == float(z["gap"])


def test_residual_rejects_inadmissible():
    g = Grid((6, 6), (1.0, 1.0), BoundaryCondition.NEUMANN)
    u = np.full((6, 6), 0.5)
    v = np.zeros((6, 6))
    prob = StepProblem.create(g, PARAMS, st(g, u, v), 1e-3)
    u2 = u.copy()
    u2[0, 0] = 1.0 - 1e-14
    with pytest.raises(InadmissibleStateError):
        residual_vector(prob, st(g, u2, v))
    u2[0, 0] = np.nan
    assert not is_admissible(st(g, u2, v))


@pytest.mark.parametrize("bc", [BoundaryCondition.PERIODIC, BoundaryCondition.NEUMANN])
def test_uniform_state_is_a_fixed_point(bc):
    # test_scheme.py:167-172 (uniform u, v = 0 is an exact fixed point)
    g = Grid((12, 10, 6), (1.0, 1.0, 1.0), bc)
    s = st(g, np.full(g.array_shape, 0.37), np.zeros(g.array_shape))
    prob = StepProblem.create(g, PARAMS, s, 1e-2)
    F = host(residual_vector(prob, s))
    assert np.all(F == 0.0)


@pytest.mark.parametrize("bc", [BoundaryCondition.PERIODIC, BoundaryCondition.NEUMANN])
def test_residual_dt_scaling(bc, rng):
    # test_scheme.py:175-186: F(dt1) - F(dt2) = (x' - x^n)(1/dt1 - 1/dt2)
    g = Grid((8, 6, 5), (1.0, 1.0, 1.0), bc)
    uo, vo = 0.5 + rng.uniform(-0.18, 0.18, g.array_shape), rng.uniform(-0.18, 0.18, g.array_shape)
    un, vn = 0.5 + rng.uniform(-0.18, 0.18, g.array_shape), rng.uniform(-0.18, 0.18, g.array_shape)
    old, new = st(g, uo, vo), st(g, un, vn)
    f1 = host(residual_vector(StepProblem.create(g, PARAMS, old, 1e-3), new))
    f2 = host(residual_vector(StepProblem.create(g, PARAMS, old, 7e-2), new))
    du = host(new.vector) - host(old.vector)
    np.testing.assert_allclose(f1 - f2, du * (1.0 / 1e-3 - 1.0 / 7e-2), rtol=1e-12, atol=1e-12)


# --------------------------------------------------------------------------- linalg

def _schwarz_setup(tag):
    z = golden(f"schwarz_{tag}.npz")
    g = grid_of(z)
    prob = StepProblem.create(g, PARAMS, st(g, z["uo"], z["vo"]), float(z["dt"]))
    J = assemble_jacobian(prob, st(g, z["un"], z["vn"]))
    return z, g, J


@pytest.mark.parametrize("tag", ["2d_neu", "2d_per", "3d_per", "3d_neu"])
@pytest.mark.parametrize("variant", ["asm", "ras-left", "ras-right"])
@pytest.mark.parametrize("solver", ["ilu0", "ilu1", "ilu2", "lu"])
def test_schwarz_apply_matches_reference(tag, variant, solver):
    z, g, J = _schwarz_setup(tag)
    pre = SchwarzPreconditioner(partition(g, int(z["nsub"]), int(z["overlap"])), SchwarzVariant(variant),
                                SubdomainSolverSpec.from_string(solver))
    assert pre.update(J) is True
    assert pre.update(J, reuse=True) is False
    out = host(pre.apply(torch.tensor(z["r"], device=DEV)))
    ref = z[f"{variant}_{solver}"]
    assert np.max(np.abs(out - ref)) <= 1e-10 * np.max(np.abs(ref))
    # bitwise reproducible
    assert np.array_equal(out, host(pre.apply(torch.tensor(z["r"], device=DEV))))


def test_apply_before_update_raises():
    g = Grid((8, 8), (1.0, 1.0), BoundaryCondition.PERIODIC)
    pre = SchwarzPreconditioner(partition(g, 2, 1), SchwarzVariant.LEFT_RAS, SubdomainSolverSpec("ilu", 0))
    with pytest.raises(RuntimeError):
        pre.apply(torch.zeros(128, dtype=torch.float64, device=DEV))


@pytest.mark.parametrize("ortho", ["mgs", "cgs2", "dcgs2"])
def test_gmres_matches_reference(ortho):
    z = golden("gmres.npz")
    g = Grid((16, 12), (1.0, 1.0), BoundaryCondition.PERIODIC)
    prob = StepProblem.create(g, PARAMS, st(g, z["uo"], z["vo"]), 1e-3)
    J = assemble_jacobian(prob, st(g, z["un"], z["vn"]))
    pre = SchwarzPreconditioner(partition(g, 4, 1), SchwarzVariant.LEFT_RAS, SubdomainSolverSpec("ilu", 0))
    pre.update(J)
    b = torch.tensor(z["b"], device=DEV)
    res = gmres(J, b, pre, 1e-8, 1e-14, 30, 500, ortho=ortho)
    assert res.converged == bool(z["conv"]) and res.iterations == int(z["its"])
    assert np.linalg.norm(host(res.x) - z["x"]) <= 1e-9 * np.linalg.norm(z["x"])
    r5 = gmres(J.matvec, b, pre, 1e-10, 1e-14, 5, 500, ortho=ortho)
    assert r5.iterations == int(z["its5"]) and r5.converged == bool(z["conv5"])
    assert np.linalg.norm(host(r5.x) - z["x5"]) <= 1e-9 * np.linalg.norm(z["x5"])
    rn = gmres(J, b, None, 1e-8, 1e-14, 30, 60, ortho=ortho)
    assert rn.iterations == int(z["itsn"]) and rn.converged == bool(z["convn"])
    assert np.linalg.norm(host(rn.x) - z["xn"]) <= 1e-8 * np.linalg.norm(z["xn"])


# --------------------------------------------------------------------------- newton

NEWTON = {
    "a": ((12, 12), False, 1e-3, 4, 1, "ilu0", {}),
    "b": ((8, 8), False, 0.01, 2, 1, "lu", dict(reuse_factorization=False)),
    "c": ((8, 8), False, 1.0, 2, 1, "lu", dict(reuse_factorization=False)),
    "d": ((8, 8), False, 1e-2, 2, 1, "ilu0", dict(max_linear_iterations=1, gmres_restart=1)),
    "e": ((10, 8, 6), True, 1e-3, 4, 1, "ilu0", {}),
}


@pytest.mark.parametrize("tag", sorted(NEWTON))
@pytest.mark.parametrize("ortho", ["mgs", "cgs2", "dcgs2"])
def test_newton_matches_reference(tag, ortho):
    z = golden("newton.npz")
    counts, periodic, dt, nsub, ov, solver, kw = NEWTON[tag]
    bc = BoundaryCondition.PERIODIC if periodic else BoundaryCondition.NEUMANN
    g = Grid(counts, tuple(1.0 for _ in counts), bc)
    s0 = st(g, z[f"{tag}_u"], z[f"{tag}_v"])
    prob = StepProblem.create(g, PARAMS, s0, dt)
    pre = SchwarzPreconditioner(partition(g, nsub, ov), SchwarzVariant.LEFT_RAS,
                                SubdomainSolverSpec.from_string(solver))
    trace = []
    sol, rep = newton_solve(prob, s0, NewtonConfig(orthogonalization=ortho, **kw), pre, trace=trace)
    conv, nit, git, fac = (int(t) for t in z[f"{tag}_report"])
    assert rep.converged == bool(conv)
    assert rep.newton_iterations == nit
    assert abs(rep.gmres_iterations - git) <= 1
    assert rep.factorizations == fac
    assert (rep.reason or "") == str(z[f"{tag}_reason"])
    ref = z[f"{tag}_x"]
    assert np.linalg.norm(host(sol.vector) - ref) <= 1e-8 * np.linalg.norm(ref)
    assert is_admissible(sol)


# --------------------------------------------------------------------------- simulate

def _run_sim(tag, ortho="cgs2"):
    from paper_2007_04560_b200.drivers import InitialSpec, RunConfig, SolverSpec, TimeSpec, simulate
    z = golden(f"sim_{tag}.npz")
    g = grid_of(z)
    center, amp, dt, horizon, nsub, eta, max_steps = (float(t) for t in z["meta"])
    cfg = RunConfig(g, PARAMS, InitialSpec("random_uniform", center, amp, 1234),
                    TimeSpec(horizon=horizon, mode=str(z["mode"]), dt=dt, dt_min=1e-4, dt_max=10.0,
                             eta=None if eta < 0 else eta),
                    SolverSpec(preconditioner=SchwarzVariant(str(z["variant"])),
                               subdomain_solver=SubdomainSolverSpec.from_string(str(z["solver"])),
                               subdomains=int(nsub), orthogonalization=ortho))
    res = simulate(cfg, max_steps=None if max_steps < 0 else int(max_steps), device=DEV)
    return z, g, res


def _check_sim(z, g, res):
    ref = z["rows"]
    assert res.status == str(z["status"])
    got = np.array([[r.step, r.time, r.dt, r.energy, r.mass_u, r.max_abs_v, r.newton, r.gmres]
                    for r in res.history])
    assert got.shape == ref.shape
    np.testing.assert_allclose(got[:, 2], ref[:, 2], rtol=1e-10)   # accepted dt sequence
    np.testing.assert_allclose(got[:, 3], ref[:, 3], rtol=1e-10)   # energy
    np.testing.assert_allclose(got[:, 4], ref[:, 4], rtol=1e-12)   # mass
    np.testing.assert_array_equal(got[:, 6], ref[:, 6])            # Newton iterations
    assert np.all(np.abs(got[:, 7] - ref[:, 7]) <= 2)              # GMRES iterations
    assert res.controller.divergence_count == int(z["divergences"])
    u, v = res.final_state.to_numpy()
    err = np.sqrt(np.sum((u - z["u"]) ** 2 + (v - z["v"]) ** 2) / np.sum(z["u"] ** 2 + z["v"] ** 2))
    assert err <= 1e-8
    # energy monotone and mass conserved (SPEC acceptance criteria)
    e = got[:, 3]
    assert np.all(np.diff(e) <= 1e-8 * np.maximum(1.0, np.abs(e[1:])))
    # mass drift at round-off level, no worse than the reference's own drift
    ref_drift = np.max(np.abs(ref[:, 4] - ref[0, 4]))
    assert np.max(np.abs(got[:, 4] - got[0, 4])) <= max(2.0 * ref_drift, 1e-12)


@pytest.mark.parametrize("ortho", ["mgs", "cgs2", "dcgs2"])
def test_simulate_config1_matches_reference(ortho):
    _check_sim(*_run_sim("c1", ortho))


def test_simulate_adaptive_2d_with_retries_matches_reference():
    _check_sim(*_run_sim("c2small"))


def test_simulate_adaptive_3d_neumann_with_retries_matches_reference():
    _check_sim(*_run_sim("c3small"))


@pytest.mark.parametrize("tag", ["c2small", "c3small"])
def test_simulate_adaptive_lagged_cgs2_matches_reference(tag):
    """The lagged second pass (dcgs2) through adaptive runs with divergence
    retries, against the reference histories."""
    _check_sim(*_run_sim(tag, "dcgs2"))


@pytest.mark.parametrize("mode", ["group", "group4", "warp", "cta"])
@pytest.mark.parametrize("solver", ["ilu0", "ilu1"])
def test_schwarz_wide_boxes_match_oracle(mode, solver, monkeypatch):
    """Boxes whose levels are wider than a warp, with each subdomain solver
    (class-group with 8 or 4 warps per CTA, plain warp, CTA-wide) forced,
    against the oracle's scalar ILU on kron(P, 1)."""
    from oracle import acch_oracle as O
    monkeypatch.setenv("ACCH_SCHWARZ_BLOCK_SOLVER", "1" if mode == "cta" else "0")
    monkeypatch.setenv("ACCH_GROUP", "1" if mode.startswith("group") else "0")
    monkeypatch.setenv("ACCH_GROUP_WARPS", "4" if mode == "group4" else "8")
    rng = np.random.default_rng(77)
    counts = (16, 14, 12)
    g = Grid(counts, (1.0, 1.0, 1.0), BoundaryCondition.NEUMANN)
    uo, vo = 0.5 + rng.uniform(-0.1, 0.1, g.array_shape), rng.uniform(-0.1, 0.1, g.array_shape)
    un, vn = uo + rng.uniform(-0.01, 0.01, g.array_shape), vo + rng.uniform(-0.01, 0.01, g.array_shape)
    prob = StepProblem.create(g, PARAMS, st(g, uo, vo), 1e-3)
    J = assemble_jacobian(prob, st(g, un, vn))
    r = rng.standard_normal(2 * g.n_cells)
    m = O.Mesh(counts, (1.0, 1.0, 1.0), False)
    Jo = O.Step(m, O.Coeffs(), uo, vo, 1e-3).jacobian(O.pack(un, vn)).assemble()
    for nsub in (1, 2):
        pre = SchwarzPreconditioner(partition(g, nsub, 1), SchwarzVariant.LEFT_RAS,
                                    SubdomainSolverSpec.from_string(solver))
        pre.update(J)
        out = host(pre.apply(torch.tensor(r, device=DEV)))
        po = O.SchwarzOracle(O.decompose(m, nsub, 1), "ras-left", solver)
        po.update(Jo)
        ref = po.apply(r)
        assert np.max(np.abs(out - ref)) <= 1e-10 * np.max(np.abs(ref))


@pytest.mark.parametrize("variant", [SchwarzVariant.LEFT_RAS, SchwarzVariant.RIGHT_RAS, SchwarzVariant.CLASSICAL])
def test_group_solver_interior_boxes_bitwise_equal_warp_solver(variant, monkeypatch):
    """Periodic 24^3 with 3x3x3 boxes: the centre box is interior (linear
    gather through the class offset table), the others wrap (general path).
    The class-group solver must give bitwise the warp solver's result (same
    per-row operation order), and match the oracle."""
    from oracle import acch_oracle as O
    rng = np.random.default_rng(5)
    counts = (24, 24, 24)
    g = Grid(counts, (1.0, 1.0, 1.0), BoundaryCondition.PERIODIC)
    uo, vo = 0.5 + rng.uniform(-0.05, 0.05, g.array_shape), rng.uniform(-0.05, 0.05, g.array_shape)
    un, vn = uo + rng.uniform(-0.01, 0.01, g.array_shape), vo + rng.uniform(-0.01, 0.01, g.array_shape)
    prob = StepProblem.create(g, PARAMS, st(g, uo, vo), 1e-3)
    J = assemble_jacobian(prob, st(g, un, vn))
    r = torch.tensor(rng.standard_normal(2 * g.n_cells), device=DEV)
    outs = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("ACCH_GROUP", mode)
        pre = SchwarzPreconditioner(partition(g, 27, 1), variant, SubdomainSolverSpec.from_string("ilu0"))
        pre.update(J)
        outs[mode] = host(pre.apply(r))
    assert np.array_equal(outs["1"], outs["0"])
    m = O.Mesh(counts, (1.0, 1.0, 1.0), True)
    Jo = O.Step(m, O.Coeffs(), uo, vo, 1e-3).jacobian(O.pack(un, vn)).assemble_fast()
    po = O.SchwarzOracle(O.decompose(m, 27, 1), variant.value, "ilu0")
    po.update(Jo)
    ref = po.apply(host(r))
    assert np.max(np.abs(outs["1"] - ref)) <= 1e-10 * np.max(np.abs(ref))


@pytest.mark.parametrize("counts", [(4, 10), (4, 6, 8), (6, 4, 5)])
def test_schwarz_tiny_periodic_axis_matches_oracle(counts):
    """A 4-cell periodic axis puts the +-2 stencil entries on one cell: the
    factorisation must sum those Jacobian contributions (the store-only
    assembly is for classes without such duplicates)."""
    from oracle import acch_oracle as O
    rng = np.random.default_rng(31)
    g = Grid(counts, (1.0,) * len(counts), BoundaryCondition.PERIODIC)
    uo, vo = 0.5 + rng.uniform(-0.05, 0.05, g.array_shape), rng.uniform(-0.05, 0.05, g.array_shape)
    un, vn = uo + rng.uniform(-0.01, 0.01, g.array_shape), vo + rng.uniform(-0.01, 0.01, g.array_shape)
    prob = StepProblem.create(g, PARAMS, st(g, uo, vo), 1e-3)
    J = assemble_jacobian(prob, st(g, un, vn))
    r = rng.standard_normal(2 * g.n_cells)
    m = O.Mesh(counts, (1.0,) * len(counts), True)
    Jo = O.Step(m, O.Coeffs(), uo, vo, 1e-3).jacobian(O.pack(un, vn)).assemble()
    for nsub, solver in ((1, "ilu0"), (2, "ilu0"), (2, "lu")):
        pre = SchwarzPreconditioner(partition(g, nsub, 1), SchwarzVariant.LEFT_RAS,
                                    SubdomainSolverSpec.from_string(solver))
        pre.update(J)
        out = host(pre.apply(torch.tensor(r, device=DEV)))
        po = O.SchwarzOracle(O.decompose(m, nsub, 1), "ras-left", solver)
        po.update(Jo)
        ref = po.apply(r)
        assert np.max(np.abs(out - ref)) <= 1e-10 * np.max(np.abs(ref))


@pytest.mark.parametrize("solver", ["ilu0", "ilu2", "lu"])
@pytest.mark.parametrize("bc", [BoundaryCondition.PERIODIC, BoundaryCondition.NEUMANN])
@pytest.mark.parametrize("counts", [(12, 12, 12), (4, 10, 12), (16, 12)])
def test_factorisation_threads_bitwise_equal(solver, bc, counts, monkeypatch):
    """factor_kernel with 32 / 64 / 128 threads per subdomain CTA (read once
    at preconditioner creation, ACCH_FACTOR_THREADS) performs every row's
    updates in the same order -- the one-warp default in 3D, the CTA-wide
    elimination of narrow levels with long rows at 128: the factors, and so
    the applies, agree bitwise.  Unsupported values are rejected."""
    rng = np.random.default_rng(9)
    g = Grid(counts, (1.0,) * len(counts), bc)
    uo, vo = 0.5 + rng.uniform(-0.05, 0.05, g.array_shape), rng.uniform(-0.05, 0.05, g.array_shape)
    un, vn = uo + rng.uniform(-0.01, 0.01, g.array_shape), vo + rng.uniform(-0.01, 0.01, g.array_shape)
    prob = StepProblem.create(g, PARAMS, st(g, uo, vo), 1e-3)
    J = assemble_jacobian(prob, st(g, un, vn))
    r = torch.tensor(rng.standard_normal(2 * g.n_cells), device=DEV)
    outs = {}
    for nt in ("32", "64", "128"):
        monkeypatch.setenv("ACCH_FACTOR_THREADS", nt)
        pre = SchwarzPreconditioner(partition(g, 8, 1), SchwarzVariant.LEFT_RAS, SubdomainSolverSpec.from_string(solver))
        pre.update(J)
        outs[nt] = host(pre.apply(r))
    assert np.array_equal(outs["32"], outs["64"]) and np.array_equal(outs["32"], outs["128"])
    monkeypatch.setenv("ACCH_FACTOR_THREADS", "256")
    with pytest.raises(ValueError):
        SchwarzPreconditioner(partition(g, 8, 1), SchwarzVariant.LEFT_RAS, SubdomainSolverSpec("ilu", 0)).update(J)


# --------------------------------------------------------------------------- warp-wide rows (exact LU)

@pytest.mark.parametrize("solver_mode", ["1", "0"])   # ACCH_GROUP: class-group solver / warp solver
@pytest.mark.parametrize("bc", [BoundaryCondition.PERIODIC, BoundaryCondition.NEUMANN])
def test_lu_wide_rows_match_oracle(bc, solver_mode, monkeypatch):
    """Exact LU on 18x18-cell extended boxes (config 2's box shape): the
    factor's levels are single rows of up to ~40 blocks, which the group solver sweeps warp-wide (one
    memory round trip per row).  Against the oracle's LU and against the
    lane-per-row sweep (ACCH_WIDE_ROWS=0)."""
    from oracle import acch_oracle as O
    rng = np.random.default_rng(11)
    counts = (64, 64)
    g = Grid(counts, (1.0, 1.0), bc)
    uo, vo = 0.5 + rng.uniform(-0.05, 0.05, g.array_shape), rng.uniform(-0.05, 0.05, g.array_shape)
    un, vn = uo + rng.uniform(-0.01, 0.01, g.array_shape), vo + rng.uniform(-0.01, 0.01, g.array_shape)
    prob = StepProblem.create(g, PARAMS, st(g, uo, vo), 1e-3)
    J = assemble_jacobian(prob, st(g, un, vn))
    r = torch.tensor(rng.standard_normal(2 * g.n_cells), device=DEV)
    monkeypatch.setenv("ACCH_GROUP", solver_mode)
    outs = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("ACCH_WIDE_ROWS", mode)
        pre = SchwarzPreconditioner(partition(g, 16, 1), SchwarzVariant.LEFT_RAS,
                                    SubdomainSolverSpec.from_string("lu"))
        pre.update(J)
        outs[mode] = host(pre.apply(r))
    m = O.Mesh(counts, (1.0, 1.0), bc == BoundaryCondition.PERIODIC)
    Jo = O.Step(m, O.Coeffs(), uo, vo, 1e-3).jacobian(O.pack(un, vn)).assemble_fast()
    po = O.SchwarzOracle(O.decompose(m, 16, 1), "ras-left", "lu")
    po.update(Jo)
    ref = po.apply(host(r))
    scale = np.max(np.abs(ref))
    assert np.max(np.abs(outs["1"] - ref)) <= 1e-10 * scale
    assert np.max(np.abs(outs["1"] - outs["0"])) <= 1e-12 * scale


@pytest.mark.parametrize("solver_mode", ["1", "0"])   # ACCH_GROUP: class-group solver / warp solver
@pytest.mark.parametrize("variant", [SchwarzVariant.LEFT_RAS, SchwarzVariant.RIGHT_RAS])
def test_ilu2_wide_rows_3d_match_oracle(variant, solver_mode, monkeypatch):
    """ILU(2) on 8^3-cell boxes of a 16^3 Neumann grid (config 3's solver):
    factor rows of up to ~90 blocks in levels of <= 4 rows, swept warp-wide
    by the warp solver (the class image is too large for the group solver)."""
    from oracle import acch_oracle as O
    rng = np.random.default_rng(12)
    counts = (16, 16, 16)
    g = Grid(counts, (1.0, 1.0, 1.0), BoundaryCondition.NEUMANN)
    uo, vo = 0.5 + rng.uniform(-0.05, 0.05, g.array_shape), rng.uniform(-0.05, 0.05, g.array_shape)
    un, vn = uo + rng.uniform(-0.01, 0.01, g.array_shape), vo + rng.uniform(-0.01, 0.01, g.array_shape)
    prob = StepProblem.create(g, PARAMS, st(g, uo, vo), 1e-3)
    J = assemble_jacobian(prob, st(g, un, vn))
    r = torch.tensor(rng.standard_normal(2 * g.n_cells), device=DEV)
    monkeypatch.setenv("ACCH_GROUP", solver_mode)
    outs = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("ACCH_WIDE_ROWS", mode)
        pre = SchwarzPreconditioner(partition(g, 8, 1), variant, SubdomainSolverSpec.from_string("ilu2"))
        pre.update(J)
        outs[mode] = host(pre.apply(r))
    m = O.Mesh(counts, (1.0, 1.0, 1.0), False)
    Jo = O.Step(m, O.Coeffs(), uo, vo, 1e-3).jacobian(O.pack(un, vn)).assemble_fast()
    po = O.SchwarzOracle(O.decompose(m, 8, 1), variant.value, "ilu2")
    po.update(Jo)
    ref = po.apply(host(r))
    scale = np.max(np.abs(ref))
    assert np.max(np.abs(outs["1"] - ref)) <= 1e-10 * scale
    assert np.max(np.abs(outs["1"] - outs["0"])) <= 1e-12 * scale


@pytest.mark.parametrize("narrow", ["1", "0"])   # ACCH_NARROW: column-sweep solver / level-wide sweeps
@pytest.mark.parametrize("variant", [SchwarzVariant.CLASSICAL, SchwarzVariant.LEFT_RAS, SchwarzVariant.RIGHT_RAS])
@pytest.mark.parametrize("case", [("lu", (48, 40), 16, BoundaryCondition.PERIODIC),
                                  ("lu", (32, 32), 16, BoundaryCondition.NEUMANN),
                                  ("ilu2", (16, 16, 16), 8, BoundaryCondition.PERIODIC),
                                  ("ilu2", (16, 8, 12), 8, BoundaryCondition.NEUMANN),
                                  ("ilu1", (16, 16, 8), 8, BoundaryCondition.NEUMANN)])
def test_narrow_classes_column_solver_matches_oracle(case, variant, narrow, monkeypatch):
    """Exact LU and ILU(k >= 1): every level of every class is at most 8 rows
    wide, so the default solver is apply_cols_kernel (column-major factors
    streamed by TMA into a shared-memory ring, column sweeps; clipped and
    wrapped boxes, all three Schwarz variants).  ACCH_NARROW=0 keeps the
    level-major layout and the warp-wide level sweeps.  Both against the
    oracle and against each other."""
    from oracle import acch_oracle as O
    solver, counts, nsub_edge, bc = case
    rng = np.random.default_rng(13)
    g = Grid(counts, (1.0,) * len(counts), bc)
    uo, vo = 0.5 + rng.uniform(-0.05, 0.05, g.array_shape), rng.uniform(-0.05, 0.05, g.array_shape)
    un, vn = uo + rng.uniform(-0.01, 0.01, g.array_shape), vo + rng.uniform(-0.01, 0.01, g.array_shape)
    prob = StepProblem.create(g, PARAMS, st(g, uo, vo), 1e-3)
    J = assemble_jacobian(prob, st(g, un, vn))
    r = torch.tensor(rng.standard_normal(2 * g.n_cells), device=DEV)
    nsub = int(np.prod([max(1, c // nsub_edge) for c in counts]))
    monkeypatch.setenv("ACCH_NARROW", narrow)
    pre = SchwarzPreconditioner(partition(g, nsub, 1), variant, SubdomainSolverSpec.from_string(solver))
    pre.update(J)
    out = host(pre.apply(r))
    out2 = host(pre.apply(r))
    assert np.array_equal(out, out2)            # run-to-run reproducible
    m = O.Mesh(counts, (1.0,) * len(counts), bc == BoundaryCondition.PERIODIC)
    Jo = O.Step(m, O.Coeffs(), uo, vo, 1e-3).jacobian(O.pack(un, vn)).assemble_fast()
    po = O.SchwarzOracle(O.decompose(m, nsub, 1), variant.value, solver)
    po.update(Jo)
    ref = po.apply(host(r))
    scale = np.max(np.abs(ref))
    assert np.max(np.abs(out - ref)) <= 1e-10 * scale
