"""Run BASELINE.json configs 1-4 through the public driver API on one B200 and
record the per-step trace the reference's `simulate` writes (step, t, dt,
energy, mass, max|v|, Newton, GMRES; drivers.py:62-73, drivers.py:118-167),
then check the two acceptance properties the paper and SPEC name: the
discrete energy is non-increasing (within 1e-8 max(1,|E|)) and
the mass <u> is conserved to round-off.

Solver settings the reference needs to converge on these grids (SURVEY.md
§8d): config 2 uses exact LU on 16x16-cell boxes, config 3 ILU(2) on 8^3-cell
boxes (ILU(0) stalls there in the reference).

Usage: python tools/run_configs.py [--configs 1,2,3] [--wall S] [--out DIR]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2007_04560_b200.drivers import (InitialSpec, RunConfig, SolverSpec, Stepper, TimeSpec,  # noqa: E402
                                           build_initial_state)
from paper_2007_04560_b200.grid import Grid  # noqa: E402
from paper_2007_04560_b200.linalg import SchwarzVariant, SubdomainSolverSpec  # noqa: E402
from paper_2007_04560_b200.physics import DEFAULT_PARAMS, diagnostics  # noqa: E402


def configs():
    ras = SchwarzVariant.LEFT_RAS
    return {
        1: ("2D 64^2 periodic, fixed dt=1e-4, 10 steps, RAS 2x2 ilu0",
            RunConfig(Grid((64, 64), (1.0, 1.0), "periodic"), DEFAULT_PARAMS, InitialSpec("random_uniform", 0.5, 0.05, 1234),
                      TimeSpec(horizon=1e-3, mode="fixed", dt=1e-4),
                      SolverSpec(ras, 1, SubdomainSolverSpec("ilu", 0), subdomains=4)), 10),
        2: ("2D 512^2 periodic, adaptive dt [1e-4,10] eta=1e4, 200 steps, RAS 16x16-cell boxes (1024) lu",
            RunConfig(Grid((512, 512), (1.0, 1.0), "periodic"), DEFAULT_PARAMS,
                      InitialSpec("random_uniform", 0.4, 0.02, 1234), TimeSpec(horizon=1e9),
                      SolverSpec(ras, 1, SubdomainSolverSpec("lu"), subdomains=1024)), 200),
        3: ("3D 128^3 Neumann, adaptive dt eta=1e2, 50 steps, GMRES(30), RAS 8^3-cell boxes (4096) ilu2",
            RunConfig(Grid((128, 128, 128), (1.0, 1.0, 1.0), "neumann"), DEFAULT_PARAMS,
                      InitialSpec("random_uniform", 0.5, 0.01, 1234), TimeSpec(horizon=1e9),
                      SolverSpec(ras, 1, SubdomainSolverSpec("ilu", 2), subdomains=4096, gmres_restart=30)), 50),
        4: ("3D 256^3 periodic, adaptive dt eta=1e2, 20 steps, GMRES(30), RAS 8^3-cell boxes (32768) ilu0 (the bench workload)",
            RunConfig(Grid((256, 256, 256), (1.0, 1.0, 1.0), "periodic"), DEFAULT_PARAMS,
                      InitialSpec("random_uniform", 0.5, 0.01, 1234), TimeSpec(horizon=1e9),
                      SolverSpec(ras, 1, SubdomainSolverSpec("ilu", 0), subdomains=32768, gmres_restart=30)), 20),
    }


def run(tag, desc, cfg, steps, wall_cap, profile=False):
    dev = torch.device("cuda", 0)
    state = build_initial_state(cfg, dev)
    e0, m0, v0 = diagnostics(state, cfg.params)
    rows = [dict(step=0, t=0.0, dt=0.0, energy=e0, mass=m0, max_abs_v=v0, newton=0, gmres=0, wall_s=0.0)]
    st = Stepper(cfg, state)
    if profile:
        st.ctx.profile(True)
        st.ctx.profile_read()
    torch.cuda.synchronize()
    t_start = time.perf_counter()
    status = "completed"
    while st.step < steps:
        w0 = time.perf_counter()
        try:
            dt, nn, ng = st.advance()
        except Exception as exc:  # stall: record and stop
            status = f"stopped: {type(exc).__name__}: {exc}"
            break
        e, m, v = diagnostics(st.state, cfg.params)
        rows.append(dict(step=st.step, t=st.t, dt=dt, energy=e, mass=m, max_abs_v=v, newton=nn, gmres=ng,
                         wall_s=time.perf_counter() - w0))
        if time.perf_counter() - t_start > wall_cap:
            status = f"wall cap {wall_cap:.0f}s reached"
            break
    torch.cuda.synchronize()
    wall = time.perf_counter() - t_start
    prof = None
    if profile:
        prof = {k: {"ms": round(v[0], 3), "launches": int(v[1])} for k, v in st.ctx.profile_read().items() if v[1]}
        st.ctx.profile(False)
    energies = [r["energy"] for r in rows]
    masses = [r["mass"] for r in rows]
    rises = [energies[i + 1] - energies[i] for i in range(len(energies) - 1)]
    tol = [1e-8 * max(1.0, abs(energies[i])) for i in range(len(energies) - 1)]
    out = dict(config=tag, workload=desc, status=status, accepted_steps=st.step, wall_s=wall,
               steps_per_s=st.step / wall if wall > 0 else None,
               newton=sum(r["newton"] for r in rows), gmres=sum(r["gmres"] for r in rows),
               retries=len(st.events), factorizations=st.factorizations,
               energy_monotone=all(d <= t for d, t in zip(rises, tol)),
               max_energy_rise=max(rises) if rises else 0.0,
               mass_drift=max(abs(m - masses[0]) for m in masses),
               energy_first=energies[0], energy_last=energies[-1], rows=rows,
               events=[list(map(str, e)) for e in st.events], kernel_ms=prof)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3")
    ap.add_argument("--wall", type=float, default=900.0, help="wall-clock cap per config (s)")
    ap.add_argument("--out", default="gpurun_out")
    ap.add_argument("--steps", type=int, default=0, help="override the step count")
    ap.add_argument("--profile", action="store_true", help="CUDA-event time per kernel category")
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    table = configs()
    for c in [int(x) for x in a.configs.split(",")]:
        desc, cfg, steps = table[c]
        res = run(c, desc, cfg, a.steps or steps, a.wall, a.profile)
        with open(os.path.join(a.out, f"config{c}_trace.json"), "w") as f:
            json.dump(res, f, indent=1)
        print(json.dumps({k: v for k, v in res.items() if k not in ("rows",)}), flush=True)


if __name__ == "__main__":
    main()
