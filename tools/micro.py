"""Kernel microbenchmarks at BASELINE sizes (CUDA-event timed, inputs > L2).

    python tools/micro.py [--n 256] [--box 8] [--reps 10]

Times: residual, Jacobian matvec, Schwarz factor / apply, GMRES vector kernels
(through one short GMRES solve with the in-library profile)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2007_04560_b200 import _native as nat  # noqa: E402
from paper_2007_04560_b200.drivers import InitialSpec, RunConfig, SolverSpec, TimeSpec, build_initial_state  # noqa
from paper_2007_04560_b200.grid import BoundaryCondition, Grid  # noqa: E402
from paper_2007_04560_b200.linalg import (SchwarzPreconditioner, SchwarzVariant, SubdomainSolverSpec,  # noqa: E402
                                          gmres, partition)
from paper_2007_04560_b200.physics import Params, State  # noqa: E402
from paper_2007_04560_b200.scheme import StepProblem, assemble_jacobian  # noqa: E402


def timeit(fn, reps):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--dim", type=int, default=3)
    ap.add_argument("--box", type=int, default=8)
    ap.add_argument("--solver", default="ilu0")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--dt", type=float, default=1e-3)
    ap.add_argument("--shape", default="", help="nx,ny,nz instead of n^dim (e.g. 512,512,64: one z-slab of config 5 on 8 GPUs)")
    args = ap.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    dev = torch.device("cuda", 0)
    counts = tuple(int(c) for c in args.shape.split(",")) if args.shape else (args.n,) * args.dim
    args.dim = len(counts)
    grid = Grid(counts, tuple(c / max(counts) for c in counts), BoundaryCondition.PERIODIC)
    params = Params(4.0, 2.0, 0.005, 0.1, 0.001)
    cfg = RunConfig(grid, params, InitialSpec("random_uniform", 0.5, 0.01, 1234), TimeSpec(1.0))
    st = build_initial_state(cfg, dev)
    N = grid.n_cells
    prob = StepProblem.create(grid, params, st, args.dt)
    g = torch.Generator(device=dev).manual_seed(1)
    x = st.vector + 1e-4 * torch.randn(2 * N, dtype=torch.float64, device=dev, generator=g)
    J = assemble_jacobian(prob, State(grid, x))
    w = torch.randn(2 * N, dtype=torch.float64, device=dev, generator=g)
    y = torch.empty_like(w)
    F = torch.empty_like(w)
    out = {}
    import ctypes
    t = timeit(lambda: nat.lib().acch_residual(prob.ctx.bind(), nat.ptr(prob.old.x), prob.dt, nat.ptr(x),
                                               nat.ptr(F), None, None), args.reps)
    out["residual"] = {"ms": t, "GB/s": 48 * N / t / 1e6, "frac": 48 * N / t / 1e6 / peak}
    t = timeit(lambda: J.matvec_into(w, y), args.reps)
    out["matvec"] = {"ms": t, "GB/s": 88 * N / t / 1e6, "frac": 88 * N / t / 1e6 / peak, "GDOF/s": 2 * N / t / 1e6}
    nsub = 1
    for c in counts:
        nsub *= c // args.box
    pre = SchwarzPreconditioner(partition(grid, nsub, 1), SchwarzVariant.LEFT_RAS,
                                SubdomainSolverSpec.from_string(args.solver))
    t = timeit(lambda: pre.update(J), 3)
    info = pre.info()
    out["factor"] = {"ms": t}
    prob.ctx.profile(True)
    prob.ctx.profile_read()
    t = timeit(lambda: pre.apply_into(w, y), args.reps)
    prof = prob.ctx.profile_read()
    ms, cnt, nb = prof["precond_apply"]
    out["apply"] = {"ms": t, "alg_GB": nb / cnt / 1e9, "GB/s": nb / cnt / t / 1e6, "frac": nb / cnt / t / 1e6 / peak,
                    "factor_bytes": info["factor_bytes"], "classes": info["classes"]}
    r = gmres(J, w, pre, 1e-8, 1e-14, 30, 60)
    prof = prob.ctx.profile_read()
    out["gmres60"] = {"iterations": r.iterations,
                      **{k: {"ms": round(v[0], 2), "n": v[1], "GB/s": round(v[2] / v[0] / 1e6, 1) if v[0] else 0}
                         for k, v in prof.items() if v[1]}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
