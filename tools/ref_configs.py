"""BASELINE.md section 3, configs 2 and 3 on the GPU box's HOST: the first K
accepted steps of the unmodified reference (baseline/_ref) with the pinned
solver settings both sides use -- config 2: 512^2 periodic, 16x16-cell boxes,
exact LU; config 3: 128^3 Neumann, 8^3-cell boxes, ILU(2); "4": the bench
workload (config 4's solver: periodic, 8^3-cell boxes, ILU(0)) at 128^3, the
largest size the reference fits in host memory -- reported as
s/step next to the GPU path's own first K steps of the same run.

    python tools/ref_configs.py [--configs 2] [--steps 3] [--threads T] [--gpu]

--gpu also runs the same K steps through paper_2007_04560_b200 on cuda:0 and
compares the accepted dt sequence and Newton counts."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def reference_run(cfg_id, steps, threads):
    assert bench.import_reference() is not None, "baseline/_ref is missing"
    from acch.cli.config import InitialSpec, RunConfig, SolverSpec, TimeSpec
    from acch.cli.drivers import simulate
    from acch.grid import BoundaryCondition, Grid
    from acch.linalg import SchwarzVariant, SubdomainSolverSpec
    from acch.physics import Params
    P = Params(4.0, 2.0, 0.005, 0.1, 0.001)
    if cfg_id == 2:
        cfg = RunConfig(Grid((512, 512), (1.0, 1.0), BoundaryCondition.PERIODIC), P,
                        InitialSpec("random_uniform", 0.4, 0.02, 1234), TimeSpec(horizon=1e9),
                        SolverSpec(SchwarzVariant.LEFT_RAS, 1, SubdomainSolverSpec("lu"), subdomains=1024))
    elif cfg_id == 4:
        # the bench workload (BASELINE config 4's solver) at 128^3 -- 256^3 needs ~160 GB in the reference
        cfg = RunConfig(Grid((128, 128, 128), (1.0, 1.0, 1.0), BoundaryCondition.PERIODIC), P,
                        InitialSpec("random_uniform", 0.5, 0.01, 1234), TimeSpec(horizon=1e9),
                        SolverSpec(SchwarzVariant.LEFT_RAS, 1, SubdomainSolverSpec("ilu", 0), subdomains=4096,
                                   gmres_restart=30))
    else:
        cfg = RunConfig(Grid((128, 128, 128), (1.0, 1.0, 1.0), BoundaryCondition.NEUMANN), P,
                        InitialSpec("random_uniform", 0.5, 0.01, 1234), TimeSpec(horizon=1e9),
                        SolverSpec(SchwarzVariant.LEFT_RAS, 1, SubdomainSolverSpec("ilu", 2), subdomains=4096,
                                   gmres_restart=30))
    t0 = time.perf_counter()
    res = simulate(cfg, threads=threads, max_steps=steps)
    t = time.perf_counter() - t0
    rows = res.history[1:]
    return {"steps": len(rows), "wall_s": t, "s_per_step": t / max(len(rows), 1), "threads": threads,
            "dt": [r.dt for r in rows], "newton": [r.newton for r in rows],
            "gmres": [r.gmres for r in rows], "energy": [r.energy for r in rows]}


def gpu_run(cfg_id, steps):
    import torch
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from run_configs import configs
    from paper_2007_04560_b200.drivers import Stepper, build_initial_state
    from paper_2007_04560_b200.physics import diagnostics
    if cfg_id == 4:
        from paper_2007_04560_b200.drivers import InitialSpec, RunConfig, SolverSpec, TimeSpec
        from paper_2007_04560_b200.grid import Grid
        from paper_2007_04560_b200.linalg import SchwarzVariant, SubdomainSolverSpec
        from paper_2007_04560_b200.physics import DEFAULT_PARAMS
        cfg = RunConfig(Grid((128, 128, 128), (1.0, 1.0, 1.0), "periodic"), DEFAULT_PARAMS,
                        InitialSpec("random_uniform", 0.5, 0.01, 1234), TimeSpec(horizon=1e9),
                        SolverSpec(SchwarzVariant.LEFT_RAS, 1, SubdomainSolverSpec("ilu", 0), subdomains=4096,
                                   gmres_restart=30))
    else:
        _, cfg, _ = configs()[cfg_id]
    dev = torch.device("cuda", 0)
    st = Stepper(cfg, build_initial_state(cfg, dev))
    out = {"dt": [], "newton": [], "gmres": [], "energy": []}
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        dt, nn, ng = st.advance()
        out["dt"].append(dt)
        out["newton"].append(nn)
        out["gmres"].append(ng)
        out["energy"].append(diagnostics(st.state, cfg.params)[0])
    torch.cuda.synchronize()
    out["wall_s"] = time.perf_counter() - t0
    out["s_per_step"] = out["wall_s"] / steps
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--threads", type=int, default=len(os.sched_getaffinity(0)))
    ap.add_argument("--gpu", action="store_true")
    a = ap.parse_args()
    for c in [int(x) for x in a.configs.split(",")]:
        line = {"config": c, "reference": reference_run(c, a.steps, a.threads)}
        if a.gpu:
            g = gpu_run(c, a.steps)
            r = line["reference"]
            line["gpu"] = g
            line["speedup"] = r["s_per_step"] / g["s_per_step"]
            line["dt_rel_diff"] = max(abs(x - y) / y for x, y in zip(g["dt"], r["dt"]))
            line["newton_equal"] = g["newton"] == r["newton"]
            line["gmres_diff"] = [x - y for x, y in zip(g["gmres"], r["gmres"])]
            line["energy_rel_diff"] = max(abs(x - y) / abs(y) for x, y in zip(g["energy"], r["energy"]))
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
