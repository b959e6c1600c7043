"""Stencil-kernel microbenchmark: residual and every Jacobian-matvec form at
256^3 (CUDA-event timed, inputs > L2), with cross-form agreement.

    python tools/mv_bench.py [--n 256] [--bc periodic|neumann] [--reps 20]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2007_04560_b200 import _native as nat  # noqa: E402
from paper_2007_04560_b200.drivers import InitialSpec, RunConfig, TimeSpec, build_initial_state  # noqa: E402
from paper_2007_04560_b200.grid import BoundaryCondition, Grid  # noqa: E402
from paper_2007_04560_b200.physics import Params, State  # noqa: E402
from paper_2007_04560_b200.scheme import StepProblem, assemble_jacobian  # noqa: E402


def timeit(fn, reps):
    for _ in range(3):
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
    ap.add_argument("--bc", default="periodic")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--forms", default="zm,twopass,fused")
    ap.add_argument("--residual", default="zm,ring")
    args = ap.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    dev = torch.device("cuda", 0)
    bc = BoundaryCondition.PERIODIC if args.bc == "periodic" else BoundaryCondition.NEUMANN
    grid = Grid((args.n,) * 3, (1.0,) * 3, bc)
    params = Params(4.0, 2.0, 0.005, 0.1, 0.001)
    cfg = RunConfig(grid, params, InitialSpec("random_uniform", 0.5, 0.01, 1234), TimeSpec(1.0))
    st = build_initial_state(cfg, dev)
    N = grid.n_cells
    prob = StepProblem.create(grid, params, st, 1e-3)
    g = torch.Generator(device=dev).manual_seed(1)
    x = st.vector + 1e-4 * torch.randn(2 * N, dtype=torch.float64, device=dev, generator=g)
    J = assemble_jacobian(prob, State(grid, x))
    w = torch.randn(2 * N, dtype=torch.float64, device=dev, generator=g)
    F = torch.empty_like(w)
    out = {"n": args.n, "bc": args.bc, "peak_gbs": peak}
    Fs = {}
    for rform in args.residual.split(","):
        name, *opt = rform.split(":")
        os.environ["ACCH_RESIDUAL"] = name
        if opt:
            os.environ["ACCH_RES_MINB"] = opt[0]
        else:
            os.environ.pop("ACCH_RES_MINB", None)
        Fr = torch.empty_like(w)
        t = timeit(lambda: nat.lib().acch_residual(prob.ctx.bind(), nat.ptr(prob.old.x), prob.dt, nat.ptr(x),
                                                   nat.ptr(Fr), None, None), args.reps)
        Fs[rform] = Fr
        out["residual_" + rform] = {"ms": round(t, 4), "frac": round(48 * N / t / 1e6 / peak, 4)}
    r0 = Fs[list(Fs)[-1]]
    out["residual_max_rel_diff"] = {f: (Fs[f] - r0).abs().max().item() / r0.abs().max().item() for f in Fs}
    os.environ.pop("ACCH_RESIDUAL", None)
    ys = {}
    for form in args.forms.split(","):
        # form[:minb[:pfd]]
        name, *opt = form.split(":")
        os.environ["ACCH_MATVEC"] = name
        for key, val in zip(("ACCH_ZM_MINB", "ACCH_ZM_PFD"), opt + [""] * 2):
            if val:
                os.environ[key] = val
            else:
                os.environ.pop(key, None)
        y = torch.empty_like(w)
        t = timeit(lambda: J.matvec_into(w, y), args.reps)
        ys[form] = y
        out["matvec_" + form] = {"ms": round(t, 4), "frac": round(88 * N / t / 1e6 / peak, 4),
                                 "GDOF/s": round(2 * N / t / 1e6, 2)}
    forms = list(ys)
    ref = ys["twopass"] if "twopass" in ys else ys[forms[0]]
    scale = ref.abs().max().item()
    out["max_rel_diff_vs_twopass"] = {f: (ys[f] - ref).abs().max().item() / scale for f in forms}
    os.environ.pop("ACCH_MATVEC", None)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
