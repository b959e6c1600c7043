"""GPU: the in-library NCCL data plane (csrc/comm.cu) on the z-slab path.

One process, one GPU: the slab grid has one rank, so NCCL's ghost-plane
exchange is a send to / receive from itself through the periodic wrap (and
nothing at Neumann walls), and its all-reduces are copies -- but every
exchange, every device all-reduce and the N > 1 branch of the
device-resident GMRES (allreduce -> Hessenberg kernel -> lost-pass finish)
run through NCCL on the library stream exactly as with 8 ranks.  Results
must equal the undecomposed single-domain path.  (Several ranks on one GPU
cannot form an NCCL communicator; the 2-rank host logic is covered on CPU
in test_slab_host.py.)"""

import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2007_04560_b200.drivers import InitialSpec, RunConfig, SolverSpec, Stepper, TimeSpec  # noqa: E402
from paper_2007_04560_b200.drivers import build_initial_state  # noqa: E402
from paper_2007_04560_b200 import _native as nat  # noqa: E402
from paper_2007_04560_b200.grid import BoundaryCondition, Grid  # noqa: E402
from paper_2007_04560_b200.linalg import (SchwarzPreconditioner, SchwarzVariant,  # noqa: E402
                                          SubdomainSolverSpec, partition)
from paper_2007_04560_b200.newton import NewtonConfig, newton_solve  # noqa: E402
from paper_2007_04560_b200.physics import Params, State  # noqa: E402
from paper_2007_04560_b200.scheme import StepProblem, assemble_jacobian, residual_vector  # noqa: E402
from paper_2007_04560_b200.slab import NcclComm, bind_comm, split_grid  # noqa: E402

PARAMS = Params(4.0, 2.0, 0.005, 0.1, 0.001)
DEV = "cuda:0"


@pytest.fixture(scope="module")
def group():
    import torch.distributed as dist
    if not dist.is_initialized():
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    yield dist
    dist.destroy_process_group()


def nccl_slab(g):
    s = split_grid(g, 1, 0)
    bind_comm(s, NcclComm(g.periodic))
    return s


def interior_np(slab, t):
    return slab.interior(t.view(slab.n_store, 2)).cpu().numpy()


@pytest.mark.parametrize("bc", [BoundaryCondition.PERIODIC, BoundaryCondition.NEUMANN])
def test_nccl_slab_residual_matvec_apply(group, bc, rng):
    g = Grid((12, 10, 16), (1.0, 1.0, 1.0), bc)
    uo = 0.5 + rng.uniform(-0.15, 0.15, g.array_shape)
    vo = rng.uniform(-0.15, 0.15, g.array_shape)
    un, vn = uo + rng.uniform(-0.01, 0.01, g.array_shape), vo + rng.uniform(-0.01, 0.01, g.array_shape)
    w = rng.standard_normal((16, 10, 12, 2))
    prob = StepProblem.create(g, PARAMS, State.from_interior(g, uo, vo, device=DEV), 1e-3)
    new = State.from_interior(g, un, vn, device=DEV)
    F_ref = residual_vector(prob, new).cpu().numpy().reshape(-1, 2)
    J = assemble_jacobian(prob, new)
    y_ref = J.matvec(torch.tensor(w.reshape(-1), device=DEV)).cpu().numpy().reshape(-1, 2)
    pre = SchwarzPreconditioner(partition(g, 8, 1), SchwarzVariant.LEFT_RAS, SubdomainSolverSpec("ilu", 0))
    pre.update(J)
    z_ref = pre.apply(torch.tensor(w.reshape(-1), device=DEV)).cpu().numpy().reshape(-1, 2)

    s = nccl_slab(g)
    p = StepProblem.create(s, PARAMS, State.from_interior(s, uo, vo, device=DEV), 1e-3)
    assert p.ctx.comm is not None and getattr(p.ctx.comm, "native", False)
    nw = State.from_interior(s, un, vn, device=DEV)
    F = interior_np(s, residual_vector(p, nw))
    Jr = assemble_jacobian(p, nw)
    wl = torch.zeros(2 * s.n_store, dtype=torch.float64, device=DEV)
    s.interior(wl.view(s.n_store, 2))[:] = torch.tensor(w.reshape(-1, 2), device=DEV)
    y = interior_np(s, Jr.matvec(wl))
    pr = SchwarzPreconditioner(partition(s, 8, 1), SchwarzVariant.LEFT_RAS, SubdomainSolverSpec("ilu", 0))
    pr.update(Jr)
    z = interior_np(s, pr.apply(wl))
    assert np.max(np.abs(F - F_ref)) <= 1e-13 * np.max(np.abs(F_ref))
    assert np.max(np.abs(y - y_ref)) <= 1e-13 * np.max(np.abs(y_ref))
    assert np.max(np.abs(z - z_ref)) <= 1e-12 * np.max(np.abs(z_ref))
    stats = p.ctx.comm_stats()
    assert stats["nccl_calls"] > 0
    if bc is BoundaryCondition.PERIODIC:
        assert stats["halo_bytes"] > 0     # self-exchange through the wrap
    torch.cuda.synchronize()


@pytest.mark.parametrize("ortho", ["dcgs2", "cgs2"])
def test_nccl_slab_newton_matches_single_domain(group, ortho, rng):
    g = Grid((12, 10, 16), (1.0, 1.0, 1.0), BoundaryCondition.PERIODIC)
    u = 0.5 + rng.uniform(-0.1, 0.1, g.array_shape)
    v = rng.uniform(-0.1, 0.1, g.array_shape)
    cfg = NewtonConfig(orthogonalization=ortho)
    s0 = State.from_interior(g, u, v, device=DEV)
    prob = StepProblem.create(g, PARAMS, s0, 2e-3)
    pre = SchwarzPreconditioner(partition(g, 8, 1), SchwarzVariant.LEFT_RAS, SubdomainSolverSpec("ilu", 0))
    sol, rep = newton_solve(prob, s0, cfg, pre)
    assert rep.converged
    s = nccl_slab(g)
    st = State.from_interior(s, u, v, device=DEV)
    p = StepProblem.create(s, PARAMS, st, 2e-3)
    pr = SchwarzPreconditioner(partition(s, 8, 1), SchwarzVariant.LEFT_RAS, SubdomainSolverSpec("ilu", 0))
    so, rp = newton_solve(p, st, cfg, pr)
    assert rp.converged and rp.newton_iterations == rep.newton_iterations
    assert abs(rp.gmres_iterations - rep.gmres_iterations) <= 1
    x_ref = sol.vector.cpu().numpy().reshape(-1, 2)
    assert np.linalg.norm(interior_np(s, so.vector) - x_ref) <= 1e-10 * np.linalg.norm(x_ref)


def test_nccl_slab_adaptive_steps_match_single_domain(group):
    g = Grid((16, 16, 32), (1.0, 1.0, 1.0), BoundaryCondition.PERIODIC)

    def cfg_for(grid):
        return RunConfig(grid, PARAMS, InitialSpec("random_uniform", 0.5, 0.01, 1234),
                         TimeSpec(horizon=10.0, mode="adaptive"), SolverSpec(subdomains=64))

    ref = Stepper(cfg_for(g), build_initial_state(cfg_for(g), device=DEV))
    ref_steps = [ref.advance() for _ in range(3)]
    x_ref = ref.state.vector.cpu().numpy().reshape(-1, 2)
    s = nccl_slab(g)
    stp = Stepper(cfg_for(s), build_initial_state(cfg_for(s), device=DEV))
    steps = [stp.advance() for _ in range(3)]
    np.testing.assert_allclose([t[0] for t in steps], [t[0] for t in ref_steps], rtol=1e-9)
    assert [t[1] for t in steps] == [t[1] for t in ref_steps]
    x = interior_np(s, stp.state.vector)
    assert np.linalg.norm(x - x_ref) <= 1e-8 * np.linalg.norm(x_ref)
