"""Residual microbenchmark at 256^3 (CUDA events, inputs > L2) on the
microbenchmark state pair U' = U^n + eps N(0,1) (eps = 1e-4 puts
the chords in the series branch as in real Newton iterates).

    python tools/res_bench.py [--n 256] [--eps 1e-4] [--reps 20] [--once]
--once: a single launch (for ncu)."""
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
from paper_2007_04560_b200.physics import Params  # noqa: E402
from paper_2007_04560_b200.scheme import StepProblem  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--eps", type=float, default=1e-4)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--once", action="store_true")
    ap.add_argument("--neumann", action="store_true")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    bc = BoundaryCondition.NEUMANN if a.neumann else BoundaryCondition.PERIODIC
    grid = Grid((a.n,) * 3, (1.0,) * 3, bc)
    params = Params(4.0, 2.0, 0.005, 0.1, 0.001)
    st = build_initial_state(RunConfig(grid, params, InitialSpec("random_uniform", 0.5, 0.01, 1234), TimeSpec(1.0)),
                             dev)
    prob = StepProblem.create(grid, params, st, 1e-3)
    g = torch.Generator(device=dev).manual_seed(1234)
    x = st.vector + a.eps * torch.randn(st.vector.numel(), dtype=torch.float64, device=dev, generator=g)
    F = torch.empty_like(x)
    L = nat.lib()

    def run():
        nat.check(L.acch_residual(prob.ctx.bind(), nat.ptr(prob.old.x), prob.dt, nat.ptr(x), nat.ptr(F), None, None),
                  "residual")
    run()
    torch.cuda.synchronize()
    if a.once:
        run()
        torch.cuda.synchronize()
        return
    ts = []
    for _ in range(a.reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    t = ts[len(ts) // 2]
    N = grid.n_cells
    peak = 6549.1
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        pass
    print(json.dumps({"n": a.n, "eps": a.eps, "ms": t, "GB/s": 48 * N / t / 1e6, "frac": 48 * N / t / 1e6 / peak,
                      "GDOF/s": 2 * N / t / 1e6, "Fnorm": float(torch.linalg.norm(F))}))


if __name__ == "__main__":
    main()
