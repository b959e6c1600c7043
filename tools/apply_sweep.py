"""Time the Schwarz apply under several env configurations in one process
(the knobs are read when a preconditioner is created).

    python tools/apply_sweep.py "ACCH_PREFETCH_DEPTH=2" "ACCH_PREFETCH_DEPTH=8,ACCH_GROUP_WARPS=4" ...
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

from micro import timeit  # noqa: E402
from paper_2007_04560_b200.drivers import InitialSpec, RunConfig, TimeSpec, build_initial_state  # noqa: E402
from paper_2007_04560_b200.grid import BoundaryCondition, Grid  # noqa: E402
from paper_2007_04560_b200.linalg import SchwarzPreconditioner, SchwarzVariant, SubdomainSolverSpec, partition  # noqa
from paper_2007_04560_b200.physics import Params, State  # noqa: E402
from paper_2007_04560_b200.scheme import StepProblem, assemble_jacobian  # noqa: E402


def main():
    n, box = 256, 8
    dev = torch.device("cuda", 0)
    grid = Grid((n,) * 3, (1.0,) * 3, BoundaryCondition.PERIODIC)
    params = Params(4.0, 2.0, 0.005, 0.1, 0.001)
    cfg = RunConfig(grid, params, InitialSpec("random_uniform", 0.5, 0.01, 1234), TimeSpec(1.0))
    st = build_initial_state(cfg, dev)
    N = grid.n_cells
    prob = StepProblem.create(grid, params, st, 1e-3)
    g = torch.Generator(device=dev).manual_seed(1)
    x = st.vector + 1e-4 * torch.randn(2 * N, dtype=torch.float64, device=dev, generator=g)
    J = assemble_jacobian(prob, State(grid, x))
    w = torch.randn(2 * N, dtype=torch.float64, device=dev, generator=g)
    ref = None
    for spec in sys.argv[1:] or [""]:
        saved = dict(os.environ)
        for kv in filter(None, spec.split(",")):
            k, v = kv.split("=")
            os.environ[k] = v
        pre = SchwarzPreconditioner(partition(grid, (n // box) ** 3, 1), SchwarzVariant.LEFT_RAS,
                                    SubdomainSolverSpec.from_string("ilu0"))
        pre.update(J)
        y = torch.empty_like(w)
        t = timeit(lambda: pre.apply_into(w, y), 10)
        if ref is None:
            ref = y.clone()
        same = bool(torch.equal(ref, y))
        print(json.dumps({"env": spec, "apply_ms": round(t, 4), "bitwise_equal_first": same}), flush=True)
        del pre
        torch.cuda.empty_cache()
        os.environ.clear()
        os.environ.update(saved)


if __name__ == "__main__":
    main()
