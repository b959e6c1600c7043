"""Generate the golden vectors that pin the oracle (and through it the GPU path).

Runs ONLY in the build container, where the reference package is readable:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba \
        PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the UNMODIFIED reference ``acch`` and records its outputs on seeded
inputs into small ``.npz`` files next to this script.  Nothing at test time
(CPU or GPU) reads /root/reference; the tests read only these files.

Cases (reference entry points in brackets):
  chord.npz        entropy_chord / entropy_chord_with_deriv battery (physics.py:213-310)
  stencil_*.npz    residual_vector, assemble_jacobian (+ matvec), total_energy,
                   admissibility_gap (scheme.py:343-484, physics.py:89-331)
  partition.npz    partition() outputs (linalg.py:161-210)
  schwarz_*.npz    SchwarzPreconditioner.apply for asm / ras-left / ras-right x
                   ilu0 / ilu1 / ilu2 / lu (linalg.py:320-396)
  gmres.npz        gmres() with a left-RAS ILU(0) preconditioner (linalg.py:411-506)
  newton.npz       newton_solve reports and solutions (newton.py:102-186)
  sim_*.npz        simulate() histories and final fields (cli/drivers.py:76-184)
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from acch.grid import BoundaryCondition, Grid  # noqa: E402
from acch.linalg import (SchwarzPreconditioner, SchwarzVariant,  # noqa: E402
                         SubdomainSolverSpec, gmres, partition)
from acch.newton import NewtonConfig, newton_solve  # noqa: E402
from acch.physics import (Params, State, admissibility_gap,  # noqa: E402
                          entropy_chord, entropy_chord_with_deriv, total_energy)
from acch.scheme import (StepProblem, assemble_jacobian, residual_vector,  # noqa: E402
                         vector_from_state)
from acch.cli.config import InitialSpec, RunConfig, SolverSpec, TimeSpec  # noqa: E402
from acch.cli.drivers import simulate  # noqa: E402

PARAMS = Params(alpha=4.0, beta=2.0, gamma=0.005, theta=0.1, rho=0.001)
BC = {"periodic": BoundaryCondition.PERIODIC, "neumann": BoundaryCondition.NEUMANN}


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {name} ({os.path.getsize(path) / 1024:.1f} KiB)")


def admissible(grid, rng, spread=0.18):
    u = 0.5 + rng.uniform(-spread, spread, size=grid.array_shape)
    v = rng.uniform(-spread, spread, size=grid.array_shape)
    return u, v


def chord_battery():
    rng = np.random.default_rng(11)
    b = rng.uniform(0.05, 0.95, 3000)
    # near pairs (series branch), far pairs, coincident, tiny separations
    a_near = b + rng.uniform(-0.3, 0.3, 3000) * np.minimum(b, 1 - b) * 0.4 * 2
    a_near = np.clip(a_near, 1e-3, 1 - 1e-3)
    a_far = rng.uniform(0.01, 0.99, 3000)
    b_tiny = rng.uniform(0.1, 0.9, 200)
    a_tiny = b_tiny + np.concatenate([np.full(100, 1e-16), np.full(100, 1e-9)]) * b_tiny
    a = np.concatenate([a_near, a_far, b[:200], a_tiny, [0.7, 0.6, 0.5]])
    bb = np.concatenate([b, b, b[:200], b_tiny, [0.5, 0.4, 0.1]])
    val = entropy_chord(a, bb, 10)
    v2, der = entropy_chord_with_deriv(a, bb, 10)
    assert np.array_equal(val, v2)
    save("chord.npz", a=a, b=bb, val=val, der=der)


def stencil_case(tag, counts, bc, seed, dt, spread=0.18, assemble=True):
    rng = np.random.default_rng(seed)
    grid = Grid(tuple(counts), tuple(1.0 for _ in counts), BC[bc])
    uo, vo = admissible(grid, rng, spread)
    # new iterate: a mix of near (series) and exactly-equal cells
    un = uo + rng.uniform(-0.02, 0.02, size=grid.array_shape)
    vn = vo + rng.uniform(-0.02, 0.02, size=grid.array_shape)
    flat_u = un.reshape(-1)
    flat_v = vn.reshape(-1)
    keep = rng.random(flat_u.size) < 0.1
    flat_u[keep] = uo.reshape(-1)[keep]
    flat_v[keep] = vo.reshape(-1)[keep]
    old = State.from_interior(grid, uo, vo)
    new = State.from_interior(grid, un, vn)
    prob = StepProblem.create(grid, PARAMS, old, dt)
    F = residual_vector(prob, new)
    # residual at the old state (exact chord branch everywhere)
    F0 = residual_vector(prob, old.copy())
    J = assemble_jacobian(prob, new)
    w = rng.standard_normal(2 * grid.n_cells)
    Jw = J.matvec(w)
    out = dict(counts=np.array(counts), periodic=np.array(bc == "periodic"), dt=np.array(dt),
               uo=uo, vo=vo, un=un, vn=vn, F=F, F0=F0, w=w, Jw=Jw,
               energy_old=np.array(total_energy(old, PARAMS)),
               energy_new=np.array(total_energy(new, PARAMS)),
               gap=np.array(admissibility_gap(un, vn)))
    if assemble:
        out.update(J_indptr=J.indptr, J_indices=J.indices, J_blocks=J.blocks)
    save(f"stencil_{tag}.npz", **out)


def partition_cases():
    cases = [((8, 8), "neumann", 4, 1), ((8, 8), "periodic", 4, 1), ((12, 8), "periodic", 6, 2),
             ((12, 8), "neumann", 6, 2), ((6, 4, 4), "periodic", 4, 1), ((6, 4, 4), "neumann", 4, 1),
             ((64, 64), "periodic", 4, 1), ((10, 7), "neumann", 6, 1), ((16, 16, 16), "periodic", 8, 1),
             ((9, 9, 9), "neumann", 27, 1), ((64, 64), "periodic", 3, 1)]
    rec = {}
    for n, (counts, bc, nsub, ov) in enumerate(cases):
        grid = Grid(counts, tuple(1.0 for _ in counts), BC[bc])
        dec = partition(grid, nsub, ov)
        rec[f"c{n}_meta"] = np.array(list(counts) + [0] * (3 - len(counts)) +
                                     [int(bc == "periodic"), nsub, ov, len(counts)])
        rec[f"c{n}_owned"] = np.concatenate(dec.owned_cells)
        rec[f"c{n}_owned_len"] = np.array([len(c) for c in dec.owned_cells])
        rec[f"c{n}_ext"] = np.concatenate(dec.extended_cells)
        rec[f"c{n}_ext_len"] = np.array([len(c) for c in dec.extended_cells])
        rec[f"c{n}_pos"] = np.concatenate(dec.owned_in_extended)
    rec["n_cases"] = np.array(len(cases))
    save("partition.npz", **rec)


def schwarz_case(tag, counts, bc, nsub, overlap, seed, dt=1e-3):
    rng = np.random.default_rng(seed)
    grid = Grid(tuple(counts), tuple(1.0 for _ in counts), BC[bc])
    uo, vo = admissible(grid, rng)
    un, vn = admissible(grid, rng)
    old = State.from_interior(grid, uo, vo)
    new = State.from_interior(grid, un, vn)
    prob = StepProblem.create(grid, PARAMS, old, dt)
    J = assemble_jacobian(prob, new)
    dec = partition(grid, nsub, overlap)
    r = rng.standard_normal(2 * grid.n_cells)
    out = dict(counts=np.array(counts), periodic=np.array(bc == "periodic"), dt=np.array(dt),
               nsub=np.array(nsub), overlap=np.array(overlap),
               uo=uo, vo=vo, un=un, vn=vn, r=r)
    for variant in ("asm", "ras-left", "ras-right"):
        for solver in ("ilu0", "ilu1", "ilu2", "lu"):
            pre = SchwarzPreconditioner(dec, SchwarzVariant(variant), SubdomainSolverSpec.from_string(solver))
            pre.update(J)
            out[f"{variant}_{solver}"] = pre.apply(r)
    save(f"schwarz_{tag}.npz", **out)


def gmres_case():
    rng = np.random.default_rng(5)
    grid = Grid((16, 12), (1.0, 1.0), BoundaryCondition.PERIODIC)
    uo, vo = admissible(grid, rng)
    un = uo + rng.uniform(-0.01, 0.01, grid.array_shape)
    vn = vo + rng.uniform(-0.01, 0.01, grid.array_shape)
    old = State.from_interior(grid, uo, vo)
    new = State.from_interior(grid, un, vn)
    prob = StepProblem.create(grid, PARAMS, old, 1e-3)
    J = assemble_jacobian(prob, new)
    b = -residual_vector(prob, new)
    pre = SchwarzPreconditioner(partition(grid, 4, 1), SchwarzVariant.LEFT_RAS, SubdomainSolverSpec("ilu", 0))
    pre.update(J)
    res = gmres(J.matvec, b, pre, 1e-8, 1e-14, 30, 500)
    res_short = gmres(J.matvec, b, pre, 1e-10, 1e-14, 5, 500)   # restart path
    res_none = gmres(J.matvec, b, None, 1e-8, 1e-14, 30, 60)    # iteration cap, no precond
    save("gmres.npz", uo=uo, vo=vo, un=un, vn=vn, b=b,
         x=res.x, its=np.array(res.iterations), conv=np.array(res.converged), rnorm=np.array(res.residual_norm),
         x5=res_short.x, its5=np.array(res_short.iterations), conv5=np.array(res_short.converged),
         xn=res_none.x, itsn=np.array(res_none.iterations), convn=np.array(res_none.converged),
         rnormn=np.array(res_none.residual_norm))


def newton_cases():
    out = {}
    specs = [  # tag, counts, bc, spread, dt, nsub, overlap, solver, cfg kwargs
        ("a", (12, 12), "neumann", 0.2, 1e-3, 4, 1, "ilu0", {}),
        ("b", (8, 8), "neumann", 0.22, 0.01, 2, 1, "lu", dict(reuse_factorization=False)),
        ("c", (8, 8), "neumann", 0.22, 1.0, 2, 1, "lu", dict(reuse_factorization=False)),
        ("d", (8, 8), "neumann", 0.18, 1e-2, 2, 1, "ilu0", dict(max_linear_iterations=1, gmres_restart=1)),
        ("e", (10, 8, 6), "periodic", 0.15, 1e-3, 4, 1, "ilu0", {}),
    ]
    for n, (tag, counts, bc, spread, dt, nsub, ov, solver, kw) in enumerate(specs):
        rng = np.random.default_rng(100 + n)
        grid = Grid(counts, tuple(1.0 for _ in counts), BC[bc])
        u, v = admissible(grid, rng, spread)
        old = State.from_interior(grid, u, v)
        prob = StepProblem.create(grid, PARAMS, old, dt)
        pre = SchwarzPreconditioner(partition(grid, nsub, ov), SchwarzVariant.LEFT_RAS,
                                    SubdomainSolverSpec.from_string(solver))
        trace = []
        sol, rep = newton_solve(prob, old.copy(), NewtonConfig(**kw), pre, trace=trace)
        out[f"{tag}_u"] = u
        out[f"{tag}_v"] = v
        out[f"{tag}_x"] = vector_from_state(sol)
        out[f"{tag}_trace"] = np.array(trace)
        out[f"{tag}_report"] = np.array([rep.converged, rep.newton_iterations, rep.gmres_iterations,
                                         rep.factorizations], dtype=np.int64)
        out[f"{tag}_reason"] = np.array(rep.reason or "")
        out[f"{tag}_fnorm"] = np.array(rep.residual_norm)
    save("newton.npz", **out)


def sim_case(tag, counts, bc, center, amp, mode, dt, horizon, nsub, solver="ilu0", eta=None,
             max_steps=None, variant="ras-left", length=1.0):
    grid = Grid(counts, tuple(length for _ in counts), BC[bc])
    cfg = RunConfig(
        grid, PARAMS, InitialSpec("random_uniform", center, amp, 1234),
        TimeSpec(horizon=horizon, mode=mode, dt=dt, dt_min=1e-4, dt_max=10.0, eta=eta),
        SolverSpec(preconditioner=SchwarzVariant(variant), overlap=1,
                   subdomain_solver=SubdomainSolverSpec.from_string(solver), subdomains=nsub))
    t0 = time.perf_counter()
    res = simulate(cfg, threads=1, max_steps=max_steps)
    wall = time.perf_counter() - t0
    h = res.history
    rows = np.array([[r.step, r.time, r.dt, r.energy, r.mass_u, r.max_abs_v, r.newton, r.gmres] for r in h])
    save(f"sim_{tag}.npz", rows=rows, status=np.array(res.status),
         u=res.final_state.u.interior, v=res.final_state.v.interior,
         divergences=np.array(res.controller.divergence_count), eta_final=np.array(res.controller.eta),
         factorizations=np.array(res.factorizations),
         meta=np.array([center, amp, dt, horizon, nsub, -1 if eta is None else eta,
                        -1 if max_steps is None else max_steps]),
         counts=np.array(counts), periodic=np.array(bc == "periodic"), mode=np.array(mode),
         solver=np.array(solver), variant=np.array(variant), wall=np.array(wall), length=np.array(length),
         eta=np.array(cfg.eta))
    print(f"  {tag}: {res.status}, {len(h) - 1} steps, {wall:.1f} s, divergences {res.controller.divergence_count}")


def io_case():
    """History CSV and VTK bytes written by the reference's cli/io.py."""
    import tempfile
    from acch.cli.io import HistoryRow, write_history, write_vtk
    from acch.grid import Field
    rng = np.random.default_rng(77)
    rows = [HistoryRow(k, 0.1 * k + 1e-17 * k, 1e-4 * (k + 1), 0.36 + rng.standard_normal() * 1e-3,
                       0.5 + 1e-13 * k, abs(rng.standard_normal()), 2 + k % 2, 10 * k, 1e-3 * k) for k in range(5)]
    out = {"rows": np.array([[r.step, r.time, r.dt, r.energy, r.mass_u, r.max_abs_v, r.newton, r.gmres, r.wall_s]
                             for r in rows])}
    with tempfile.TemporaryDirectory() as d:
        write_history(rows, os.path.join(d, "h.csv"))
        out["csv"] = np.array(open(os.path.join(d, "h.csv")).read())
        for tag, counts in (("2d", (7, 5)), ("3d", (5, 4, 6))):
            grid = Grid(counts, tuple(0.5 + 0.25 * a for a in range(len(counts))), BoundaryCondition.PERIODIC)
            u = 0.5 + rng.uniform(-0.2, 0.2, grid.array_shape)
            v = rng.uniform(-0.2, 0.2, grid.array_shape)
            st = State(Field.from_interior(grid, u), Field.from_interior(grid, v))
            write_vtk(st, os.path.join(d, f"{tag}.vtk"), title=f"snapshot {tag}")
            out[f"vtk_{tag}"] = np.array(open(os.path.join(d, f"{tag}.vtk")).read())
            out[f"u_{tag}"] = u
            out[f"v_{tag}"] = v
            out[f"counts_{tag}"] = np.array(counts)
            out[f"lengths_{tag}"] = np.array(grid.lengths)
    save("io.npz", **out)


def main():
    which = set(sys.argv[1:])

    def want(k):
        return not which or k in which

    if want("chord"):
        chord_battery()
    if want("io"):
        io_case()
    if want("stencil"):
        stencil_case("2d_neu", (8, 6), "neumann", 1, 1e-3)
        stencil_case("2d_per", (8, 6), "periodic", 2, 1e-3)
        stencil_case("2d_per4", (4, 4), "periodic", 3, 1e-2)
        stencil_case("3d_neu", (5, 4, 6), "neumann", 4, 1e-3)
        stencil_case("3d_per", (6, 4, 5), "periodic", 5, 1e-3)
        stencil_case("2d_per_big", (64, 48), "periodic", 6, 1e-4, spread=0.05, assemble=False)
        stencil_case("3d_neu_big", (20, 16, 12), "neumann", 7, 1e-4, spread=0.05, assemble=False)
    if want("partition"):
        partition_cases()
    if want("schwarz"):
        schwarz_case("2d_neu", (12, 10), "neumann", 4, 1, 21)
        schwarz_case("2d_per", (12, 12), "periodic", 4, 1, 22)
        schwarz_case("3d_per", (8, 6, 6), "periodic", 4, 1, 23)
        schwarz_case("3d_neu", (6, 6, 6), "neumann", 8, 1, 24)
    if want("gmres"):
        gmres_case()
    if want("newton"):
        newton_cases()
    if want("sim"):
        # BASELINE config 1: 64^2 periodic, fixed dt 1e-4, 10 steps, 2x2 left-RAS ILU(0)
        sim_case("c1", (64, 64), "periodic", 0.5, 0.05, "fixed", 1e-4, 10e-4, 4)
        # config-2 analogue at 32^2: adaptive, eta=1e4 (2D default), retries happen
        sim_case("c2small", (32, 32), "periodic", 0.4, 0.02, "adaptive", 1e-4, 10.0, 4, max_steps=40)
        # config-3 analogue: 3D Neumann, adaptive eta=1e2, 8 boxes
        sim_case("c3small", (16, 16, 16), "neumann", 0.5, 0.01, "adaptive", 1e-4, 10.0, 8, max_steps=4)
    # the BASELINE solver regimes (VERDICT r1 "next" #1)
    if want("sim3p"):
        # config-3 stiffness proxy: 32^3 Neumann on a box of side 0.25 (dx = 1/128, the
        # 128^3 grid's spacing), 8^3-cell boxes, ILU(2) (ILU(0)/ILU(1) fail here), eta = 1e2
        sim_case("c3proxy", (32, 32, 32), "neumann", 0.5, 0.01, "adaptive", 1e-4, 10.0, 64, solver="ilu2",
                 max_steps=3, length=0.25)
    if want("sim2a"):
        # config-2 analogue: 128^2 periodic, 16x16-cell boxes, exact LU, adaptive eta = 1e4
        sim_case("c2analog", (128, 128), "periodic", 0.4, 0.02, "adaptive", 1e-4, 10.0, 64, solver="lu",
                 max_steps=20)
    if want("sim4a"):
        # config-4 analogue (the bench's regime): 32^3 periodic, 8^3-cell boxes, ILU(0), eta = 1e2
        sim_case("c4analog", (32, 32, 32), "periodic", 0.5, 0.01, "adaptive", 1e-4, 10.0, 64, max_steps=5)


if __name__ == "__main__":
    main()
