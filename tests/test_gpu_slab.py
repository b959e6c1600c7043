"""GPU: the z-slab decomposition against the single-domain path.

Ranks are emulated as threads of one process on one GPU (slab.ThreadComm):
each rank owns a context, a stream, its slab with two ghost planes per side,
and meets the others only in host-side halo / allreduce hooks.  Results must
equal the undecomposed solve up to the reduction order of the dots."""

import threading

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2007_04560_b200.drivers import InitialSpec, RunConfig, SolverSpec, Stepper, TimeSpec  # noqa: E402
from paper_2007_04560_b200.drivers import build_initial_state  # noqa: E402
from paper_2007_04560_b200.grid import BoundaryCondition, Grid  # noqa: E402
from paper_2007_04560_b200.linalg import (SchwarzPreconditioner, SchwarzVariant,  # noqa: E402
                                          SubdomainSolverSpec, partition)
from paper_2007_04560_b200.newton import NewtonConfig, newton_solve  # noqa: E402
from paper_2007_04560_b200.physics import Params, State  # noqa: E402
from paper_2007_04560_b200.scheme import StepProblem, assemble_jacobian, residual_vector  # noqa: E402
from paper_2007_04560_b200.slab import ThreadGroup, bind_comm, split_grid  # noqa: E402

PARAMS = Params(4.0, 2.0, 0.005, 0.1, 0.001)
DEV = "cuda:0"


def run_ranks(grp, nranks, fn):
    out = [None] * nranks
    errs = []

    def worker(r):
        try:
            with torch.cuda.stream(torch.cuda.Stream(device=DEV)):
                out[r] = fn(r)
                torch.cuda.current_stream().synchronize()
        except BaseException as e:  # unblock the other ranks
            errs.append(e)
            grp.barrier.abort()

    ts = [threading.Thread(target=worker, args=(r,)) for r in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    if errs:
        raise errs[0]
    return out


def slabs_for(g, nranks):
    grp = ThreadGroup(nranks)
    slabs = [split_grid(g, nranks, r) for r in range(nranks)]
    for r, s in enumerate(slabs):
        bind_comm(s, grp.comm(r, g.periodic))
    return grp, slabs


def fields(g, rng, spread=0.15):
    u = 0.5 + rng.uniform(-spread, spread, g.array_shape)
    v = rng.uniform(-spread, spread, g.array_shape)
    return u, v


def interior_np(slab, t):
    """(nz_local*ny*nx, 2) interior of a stored vector as numpy."""
    return slab.interior(t.view(slab.n_store, 2)).cpu().numpy()


CASES = [((12, 10, 16), BoundaryCondition.PERIODIC, 2), ((12, 10, 16), BoundaryCondition.NEUMANN, 2),
         ((8, 8, 32), BoundaryCondition.PERIODIC, 4), ((8, 12, 24), BoundaryCondition.NEUMANN, 3)]


@pytest.mark.parametrize("counts,bc,nranks", CASES)
def test_slab_residual_and_matvec_match_single_domain(counts, bc, nranks, rng):
    g = Grid(counts, (1.0, 1.0, 1.0), bc)
    uo, vo = fields(g, rng)
    un, vn = uo + rng.uniform(-0.01, 0.01, g.array_shape), vo + rng.uniform(-0.01, 0.01, g.array_shape)
    w = rng.standard_normal((counts[2], counts[1], counts[0], 2))
    prob = StepProblem.create(g, PARAMS, State.from_interior(g, uo, vo, device=DEV), 1e-3)
    new = State.from_interior(g, un, vn, device=DEV)
    F_ref = residual_vector(prob, new).cpu().numpy().reshape(-1, 2)
    J = assemble_jacobian(prob, new)
    y_ref = J.matvec(torch.tensor(w.reshape(-1), device=DEV)).cpu().numpy().reshape(-1, 2)
    grp, slabs = slabs_for(g, nranks)

    def rank_fn(r):
        s = slabs[r]
        z0, z1 = s.z0, s.z0 + s.counts[2]
        p = StepProblem.create(s, PARAMS, State.from_interior(s, uo[z0:z1], vo[z0:z1], device=DEV), 1e-3)
        nw = State.from_interior(s, un[z0:z1], vn[z0:z1], device=DEV)
        F = residual_vector(p, nw)
        Jr = assemble_jacobian(p, nw)
        wl = torch.zeros(2 * s.n_store, dtype=torch.float64, device=DEV)
        s.interior(wl.view(s.n_store, 2))[:] = torch.tensor(w[z0:z1].reshape(-1, 2), device=DEV)
        y = Jr.matvec(wl)
        return interior_np(s, F), interior_np(s, y)

    res = run_ranks(grp, nranks, rank_fn)
    F = np.concatenate([r[0] for r in res])
    y = np.concatenate([r[1] for r in res])
    assert np.max(np.abs(F - F_ref)) <= 1e-13 * np.max(np.abs(F_ref))
    assert np.max(np.abs(y - y_ref)) <= 1e-13 * np.max(np.abs(y_ref))


@pytest.mark.parametrize("counts,bc,nranks", CASES[:2])
@pytest.mark.parametrize("solver", ["ilu0", "ilu1", "ilu2"])   # ilu2: the column-sweep solver on slab boxes
def test_slab_schwarz_apply_matches_single_domain(counts, bc, nranks, solver, rng):
    g = Grid(counts, (1.0, 1.0, 1.0), bc)
    uo, vo = fields(g, rng)
    un, vn = fields(g, rng)
    r_glob = rng.standard_normal((counts[2], counts[1], counts[0], 2))
    nsub = 8
    prob = StepProblem.create(g, PARAMS, State.from_interior(g, uo, vo, device=DEV), 1e-3)
    J = assemble_jacobian(prob, State.from_interior(g, un, vn, device=DEV))
    pre = SchwarzPreconditioner(partition(g, nsub, 1), SchwarzVariant.LEFT_RAS, SubdomainSolverSpec.from_string(solver))
    pre.update(J)
    z_ref = pre.apply(torch.tensor(r_glob.reshape(-1), device=DEV)).cpu().numpy().reshape(-1, 2)
    grp, slabs = slabs_for(g, nranks)

    def rank_fn(r):
        s = slabs[r]
        z0, z1 = s.z0, s.z0 + s.counts[2]
        p = StepProblem.create(s, PARAMS, State.from_interior(s, uo[z0:z1], vo[z0:z1], device=DEV), 1e-3)
        Jr = assemble_jacobian(p, State.from_interior(s, un[z0:z1], vn[z0:z1], device=DEV))
        pr = SchwarzPreconditioner(partition(s, nsub, 1), SchwarzVariant.LEFT_RAS,
                                   SubdomainSolverSpec.from_string(solver))
        pr.update(Jr)
        rl = torch.zeros(2 * s.n_store, dtype=torch.float64, device=DEV)
        s.interior(rl.view(s.n_store, 2))[:] = torch.tensor(r_glob[z0:z1].reshape(-1, 2), device=DEV)
        return interior_np(s, pr.apply(rl))

    z = np.concatenate(run_ranks(grp, nranks, rank_fn))
    assert np.max(np.abs(z - z_ref)) <= 1e-12 * np.max(np.abs(z_ref))


@pytest.mark.parametrize("counts,bc,nranks", CASES[:3])
def test_slab_newton_matches_single_domain(counts, bc, nranks, rng):
    g = Grid(counts, (1.0, 1.0, 1.0), bc)
    u, v = fields(g, rng, 0.1)
    nsub = 8 if nranks <= 2 else 16
    cfg = NewtonConfig()
    s0 = State.from_interior(g, u, v, device=DEV)
    prob = StepProblem.create(g, PARAMS, s0, 2e-3)
    pre = SchwarzPreconditioner(partition(g, nsub, 1), SchwarzVariant.LEFT_RAS, SubdomainSolverSpec("ilu", 0))
    sol, rep = newton_solve(prob, s0, cfg, pre)
    assert rep.converged
    x_ref = sol.vector.cpu().numpy().reshape(-1, 2)
    grp, slabs = slabs_for(g, nranks)

    def rank_fn(r):
        s = slabs[r]
        z0, z1 = s.z0, s.z0 + s.counts[2]
        st = State.from_interior(s, u[z0:z1], v[z0:z1], device=DEV)
        p = StepProblem.create(s, PARAMS, st, 2e-3)
        pr = SchwarzPreconditioner(partition(s, nsub, 1), SchwarzVariant.LEFT_RAS, SubdomainSolverSpec("ilu", 0))
        so, rp = newton_solve(p, st, cfg, pr)
        return interior_np(s, so.vector), rp

    res = run_ranks(grp, nranks, rank_fn)
    x = np.concatenate([r[0] for r in res])
    for _, rp in res:
        assert rp.converged and rp.newton_iterations == rep.newton_iterations
        assert abs(rp.gmres_iterations - rep.gmres_iterations) <= 1
    assert np.linalg.norm(x - x_ref) <= 1e-10 * np.linalg.norm(x_ref)


def test_slab_adaptive_steps_match_single_domain():
    """Three adaptive steps of a 3D periodic run: same dt sequence, same fields."""
    g = Grid((16, 16, 32), (1.0, 1.0, 1.0), BoundaryCondition.PERIODIC)
    nranks = 2

    def cfg_for(grid):
        return RunConfig(grid, PARAMS, InitialSpec("random_uniform", 0.5, 0.01, 1234),
                         TimeSpec(horizon=10.0, mode="adaptive"),
                         SolverSpec(subdomains=64, orthogonalization="cgs2"))

    ref = Stepper(cfg_for(g), build_initial_state(cfg_for(g), device=DEV))
    ref_dt = [ref.advance()[0] for _ in range(3)]
    x_ref = ref.state.vector.cpu().numpy().reshape(-1, 2)
    grp, slabs = slabs_for(g, nranks)

    def rank_fn(r):
        s = slabs[r]
        stp = Stepper(cfg_for(s), build_initial_state(cfg_for(s), device=DEV))
        dts = [stp.advance()[0] for _ in range(3)]
        return dts, interior_np(s, stp.state.vector)

    res = run_ranks(grp, nranks, rank_fn)
    for dts, _ in res:
        np.testing.assert_allclose(dts, ref_dt, rtol=1e-9)
    x = np.concatenate([r[1] for r in res])
    assert np.linalg.norm(x - x_ref) <= 1e-8 * np.linalg.norm(x_ref)
