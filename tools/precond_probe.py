"""Time one Schwarz apply / factorisation for the BASELINE config 2 and 3
preconditioners (LU on 16x16-cell boxes at 512^2; ILU(2) on 8^3-cell boxes at
128^3 Neumann) and the bench's ILU(0) at 256^3, with ACCH_DEBUG=1 printing
which solver the library picked.

    python tools/precond_probe.py [c2|c3|c4 ...] [ENV=VAL,...]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

from micro import timeit  # noqa: E402
from paper_2007_04560_b200.drivers import InitialSpec, RunConfig, TimeSpec, build_initial_state  # noqa: E402
from paper_2007_04560_b200.grid import Grid  # noqa: E402
from paper_2007_04560_b200.linalg import SchwarzPreconditioner, SchwarzVariant, SubdomainSolverSpec, partition  # noqa
from paper_2007_04560_b200.physics import DEFAULT_PARAMS, State  # noqa: E402
from paper_2007_04560_b200.scheme import StepProblem, assemble_jacobian  # noqa: E402

CASES = {"c2": ((512, 512), "periodic", 0.4, 0.02, 1024, "lu"),
         "c3": ((128, 128, 128), "neumann", 0.5, 0.01, 4096, "ilu2"),
         "c4": ((256, 256, 256), "periodic", 0.5, 0.01, 32768, "ilu0")}


def main():
    cases = [a for a in sys.argv[1:] if a in CASES] or ["c2", "c3"]
    envs = [a for a in sys.argv[1:] if a not in CASES] or [""]
    dev = torch.device("cuda", 0)
    for c in cases:
        counts, bc, cu, amp, nsub, solver = CASES[c]
        grid = Grid(counts, (1.0,) * len(counts), bc)
        cfg = RunConfig(grid, DEFAULT_PARAMS, InitialSpec("random_uniform", cu, amp, 1234), TimeSpec(1.0))
        st = build_initial_state(cfg, dev)
        n2 = 2 * grid.n_cells
        prob = StepProblem.create(grid, DEFAULT_PARAMS, st, 1e-3)
        g = torch.Generator(device=dev).manual_seed(1)
        x = st.vector + 1e-4 * torch.randn(n2, dtype=torch.float64, device=dev, generator=g)
        J = assemble_jacobian(prob, State(grid, x))
        w = torch.randn(n2, dtype=torch.float64, device=dev, generator=g)
        ref = None
        for spec in envs:
            saved = dict(os.environ)
            os.environ["ACCH_DEBUG"] = "1"
            for kv in filter(None, spec.split(",")):
                k, v = kv.split("=")
                os.environ[k] = v
            t0 = time.perf_counter()
            pre = SchwarzPreconditioner(partition(grid, nsub, 1), SchwarzVariant.LEFT_RAS,
                                        SubdomainSolverSpec.from_string(solver))
            t_setup = time.perf_counter() - t0
            t_fact = timeit(lambda: (pre.invalidate(), pre.update(J)), 3)
            y = torch.empty_like(w)
            t = timeit(lambda: pre.apply_into(w, y), 10)
            if ref is None:
                ref = y.clone()
            rel = float((y - ref).abs().max() / ref.abs().max())
            print(json.dumps({"case": c, "env": spec, "solver": solver, "subdomains": nsub,
                              "setup_s": round(t_setup, 3), "factor_ms": round(t_fact, 3),
                              "apply_ms": round(t, 4), "max_rel_diff_vs_first": rel}), flush=True)
            del pre
            torch.cuda.empty_cache()
            os.environ.clear()
            os.environ.update(saved)


if __name__ == "__main__":
    main()
