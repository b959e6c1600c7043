"""Run configuration and the accepted-step time loop (the hot path's caller:
the reference's acch/cli/config.py:23-120 dataclasses and
acch/cli/drivers.py:26-184 ``build_initial_state`` / ``simulate``).

INI parsing and the experiment drivers are out of scope; the dataclasses
keep the reference's field names and defaults so a RunConfig built for the
reference maps over field by field.  ``simulate(out_dir=...)`` writes the
reference's history CSV and VTK snapshots (io.py)."""

from __future__ import annotations

import os
import time
from dataclasses import dataclass, field, replace

import numpy as np

from .exceptions import ConfigError, SolverStallError
from .grid import Grid
from .linalg import SchwarzPreconditioner, SchwarzVariant, SubdomainSolverSpec, partition
from .newton import NewtonConfig, newton_solve
from .physics import Params, State, diagnostics
from .scheme import StepProblem
from .timestep import StepController

COMPLETED = "completed"
STALLED = "stalled"


@dataclass(frozen=True)
class InitialSpec:
    kind: str = "random_uniform"
    center_u: float = 0.55
    amplitude: float = 0.05
    seed: int = 1234

    def __post_init__(self):
        if self.kind not in ("trigonometric", "random_uniform"):
            raise ConfigError(f"unknown initial condition {self.kind!r}")
        if self.kind == "random_uniform":
            lo_u, hi_u = self.center_u - self.amplitude, self.center_u + self.amplitude
            if not (0.0 < lo_u - self.amplitude and hi_u + self.amplitude < 1.0):
                raise ConfigError("random initial condition can produce inadmissible states")


@dataclass(frozen=True)
class TimeSpec:
    horizon: float
    mode: str = "adaptive"
    dt: float = 1e-4
    dt_min: float = 1e-4
    dt_max: float = 10.0
    eta: float | None = None


@dataclass(frozen=True)
class SolverSpec:
    preconditioner: SchwarzVariant = SchwarzVariant.LEFT_RAS
    overlap: int = 1
    subdomain_solver: SubdomainSolverSpec = SubdomainSolverSpec("ilu", 0)
    reuse: bool = True
    subdomains: int = 0
    refreeze_every: int = 1
    rel_tol: float = 1e-6
    abs_tol: float = 1e-13
    lin_rel_tol: float = 1e-8
    lin_abs_tol: float = 1e-14
    max_newton: int = 50
    gmres_restart: int = 30
    max_linear_iterations: int = 500
    orthogonalization: str = "dcgs2"


@dataclass(frozen=True)
class OutputSpec:
    history: str = "history.csv"
    snapshot_times: tuple = ()
    snapshot_every: int = 0


@dataclass(frozen=True)
class RunConfig:
    grid: Grid
    params: Params
    initial: InitialSpec
    time: TimeSpec
    solver: SolverSpec = SolverSpec()
    output: OutputSpec = OutputSpec()

    @property
    def eta(self) -> float:
        if self.time.eta is not None:
            return self.time.eta
        return 1e4 if self.grid.dim == 2 else 1e2

    def make_controller(self) -> StepController:
        if self.time.mode == "fixed":
            return StepController(self.time.dt, self.time.dt, self.eta, fixed_dt=self.time.dt)
        return StepController(self.time.dt_min, self.time.dt_max, self.eta)

    def make_newton_config(self) -> NewtonConfig:
        s = self.solver
        return NewtonConfig(rel_tol=s.rel_tol, abs_tol=s.abs_tol, lin_rel_tol=s.lin_rel_tol,
                            lin_abs_tol=s.lin_abs_tol, max_iterations=s.max_newton, gmres_restart=s.gmres_restart,
                            max_linear_iterations=s.max_linear_iterations, reuse_factorization=s.reuse,
                            refactor_on_entry=s.refreeze_every <= 1, orthogonalization=s.orthogonalization)

    def with_solver(self, **kw) -> "RunConfig":
        return replace(self, solver=replace(self.solver, **kw))

    def with_time(self, **kw) -> "RunConfig":
        return replace(self, time=replace(self.time, **kw))


def initial_fields(config: RunConfig):
    """Host fields of the configured initial condition (drivers.py:26-46):
    one seeded generator, u drawn before v, reversed-axis shape, so the
    inputs are bitwise those of the reference."""
    grid = config.grid
    spec = config.initial
    if spec.kind == "trigonometric":
        if grid.dim != 2:
            raise ConfigError("trigonometric initial condition is 2D only")
        x, y = grid.center_mesh()
        sx = np.sin(2.0 * np.pi * x) ** 2
        cy = np.cos(2.0 * np.pi * y) ** 2
        return 0.4 * (sx + cy) + 0.1, 0.4 * (sx - cy)
    rng = np.random.default_rng(spec.seed)
    u = spec.center_u + rng.uniform(-spec.amplitude, spec.amplitude, grid.array_shape)
    v = rng.uniform(-spec.amplitude, spec.amplitude, grid.array_shape)
    return u, v


def build_initial_state(config: RunConfig, device=None) -> State:
    grid = config.grid
    if getattr(grid, "nz_global", 0):
        # a slab: draw the global fields (bitwise the reference's inputs) and keep this rank's planes
        from .slab import local_fields
        from dataclasses import replace as _replace
        u, v = initial_fields(_replace(config, grid=grid.global_grid()))
        u, v = local_fields(grid, u, v)
        return State.from_interior(grid, np.ascontiguousarray(u), np.ascontiguousarray(v), device=device)
    u, v = initial_fields(config)
    return State.from_interior(grid, u, v, device=device)


@dataclass
class HistoryRow:
    step: int
    time: float
    dt: float
    energy: float
    mass_u: float
    max_abs_v: float
    newton: int
    gmres: int
    wall_s: float


@dataclass
class SimulationResult:
    status: str
    history: list
    final_state: State
    controller: StepController
    factorizations: int = 0
    events: list = field(default_factory=list)

    @property
    def completed(self) -> bool:
        return self.status == COMPLETED


class Stepper:
    """The body of the reference's time loop (drivers.py:118-167), one
    accepted step per ``advance()`` call: predict dt, solve with retries
    (controller shrink + fresh factorisation on divergence), update the
    two-level history the predictor needs.  Raises SolverStallError when the
    controller gives up."""

    def __init__(self, config: RunConfig, state: State, threads: int = 1):
        self.config = config
        self.grid = config.grid
        self.state = state
        self.controller = config.make_controller()
        n_sub = config.solver.subdomains or threads
        self.decomposition = partition(self.grid, n_sub, config.solver.overlap)
        self.newton_cfg = config.make_newton_config()
        from . import _native
        self.ctx = _native.context_for(self.grid, config.params, state.device)
        self.precond = SchwarzPreconditioner(self.decomposition, config.solver.preconditioner,
                                             config.solver.subdomain_solver)
        self.t = 0.0
        self.step = 0
        self.dt_prev = None
        self.x_now = state.vector
        self.x_prev = None
        self.since = 0
        self.refreeze_every = max(1, config.solver.refreeze_every)
        self.factorizations = 0
        self.events = []

    def snapshot(self) -> dict:
        """Everything the next steps depend on (state, predictor history,
        controller gains and counters), so a run can be replayed exactly."""
        ctl = self.controller
        return {"x": self.state.x.clone(), "x_prev": None if self.x_prev is None else self.x_prev.clone(),
                "t": self.t, "step": self.step, "dt_prev": self.dt_prev, "since": self.since, "eta": ctl.eta,
                "stalled": ctl._stalled_retries, "div": ctl.divergence_count, "events": len(self.events),
                "fact": self.factorizations}

    def restore(self, snap: dict) -> None:
        ctl = self.controller
        self.state = State(self.grid, snap["x"].clone())
        self.x_now = self.state.vector
        self.x_prev = None if snap["x_prev"] is None else snap["x_prev"].clone()
        self.t, self.step, self.dt_prev, self.since = snap["t"], snap["step"], snap["dt_prev"], snap["since"]
        ctl.eta, ctl._stalled_retries, ctl.divergence_count = snap["eta"], snap["stalled"], snap["div"]
        del self.events[snap["events"]:]
        self.factorizations = snap["fact"]
        self.precond.invalidate()

    def advance(self):
        """One accepted step; returns (dt, newton iterations, gmres iterations)."""
        self.step += 1
        ctl = self.controller
        if self.step == 1 or self.x_prev is None:
            dt = ctl.initial_dt()
        else:
            dt = ctl.predict_dt(self.x_now, self.x_prev, self.dt_prev, ctx=self.ctx)
        if self.since >= self.refreeze_every:
            self.precond.invalidate()
            self.since = 0
        newton_count = gmres_count = 0
        while True:
            prob = StepProblem.create(self.grid, self.config.params, self.state, dt)
            new_state, report = newton_solve(prob, self.state, self.newton_cfg, self.precond)
            newton_count += report.newton_iterations
            gmres_count += report.gmres_iterations
            self.factorizations += report.factorizations
            if report.converged:
                break
            self.events.append((self.step, dt, report.reason))
            dt = ctl.on_divergence(dt)
            self.precond.invalidate()
            self.since = 0
        self.since += 1
        ctl.note_success()
        self.t += dt
        self.x_prev = self.x_now
        self.x_now = new_state.vector
        self.dt_prev = dt
        self.state = new_state
        return dt, newton_count, gmres_count


def simulate(config: RunConfig, threads: int = 1, out_dir: str | None = None, snapshot_every: int = 0,
             max_steps: int | None = None, state: State | None = None, device=None,
             diagnostics_every: int = 1) -> SimulationResult:
    """Advance from t = 0 to the horizon (drivers.py:76-184) and record
    energy / mass / max|v| per accepted step.  ``events`` lists
    (step, dt, reason) for every divergence.  With ``out_dir`` the history
    CSV is written incrementally (flushed per step) and VTK snapshots at the
    configured times / every ``snapshot_every`` steps plus ``final.vtk``,
    as the reference does; partial outputs survive a stall."""
    from .io import HistoryWriter, write_vtk
    if state is None:
        state = build_initial_state(config, device)
    stepper = Stepper(config, state, threads)
    history = []
    snapshot_every = snapshot_every or config.output.snapshot_every
    pending = sorted(config.output.snapshot_times)
    writer = None
    if out_dir is not None:
        os.makedirs(out_dir, exist_ok=True)
        writer = HistoryWriter(os.path.join(out_dir, config.output.history))

    def row(step, t, dt, st, newton, gm, wall):
        if diagnostics_every and (step % diagnostics_every == 0):
            e, m, v = diagnostics(st, config.params)
        else:
            e = m = v = float("nan")
        r = HistoryRow(step, t, dt, e, m, v, newton, gm, wall)
        history.append(r)
        if writer is not None:
            writer.write(r)

    row(0, 0.0, 0.0, state, 0, 0, 0.0)
    status = COMPLETED
    horizon = config.time.horizon
    try:
        while stepper.t < horizon * (1.0 - 1e-12):
            if max_steps is not None and stepper.step >= max_steps:
                break
            wall0 = time.perf_counter()
            try:
                dt, nn, ng = stepper.advance()
            except SolverStallError:
                status = STALLED
                break
            row(stepper.step, stepper.t, dt, stepper.state, nn, ng, time.perf_counter() - wall0)
            if out_dir is not None:
                t = stepper.t
                while pending and t >= pending[0] * (1.0 - 1e-12):
                    target = pending.pop(0)
                    write_vtk(stepper.state, os.path.join(out_dir, f"snapshot_t{target:g}.vtk"),
                              title=f"state at t={t:.10g} (requested {target:g})")
                if snapshot_every and stepper.step % snapshot_every == 0:
                    write_vtk(stepper.state, os.path.join(out_dir, f"step_{stepper.step:06d}.vtk"))
    finally:
        if writer is not None:
            writer.close()
    if out_dir is not None:
        write_vtk(stepper.state, os.path.join(out_dir, "final.vtk"), title="final state")
    return SimulationResult(status, history, stepper.state, stepper.controller, stepper.factorizations,
                            stepper.events)


__all__ = ["InitialSpec", "TimeSpec", "SolverSpec", "OutputSpec", "RunConfig", "initial_fields", "build_initial_state",
           "HistoryRow", "SimulationResult", "Stepper", "simulate", "COMPLETED", "STALLED"]
