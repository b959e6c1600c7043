"""CPU-only checks of the host layer and the C ABI boundary (no GPU needed)."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden

HEADER = os.path.join(ROOT, "include", "acch_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:acch_status|const char \*|int32_t|int64_t)\s*\*?\s*(acch_\w+)\s*\(",
                                 text, flags=re.M)))


def test_library_loads_and_exports_every_declared_symbol():
    from paper_2007_04560_b200 import _native
    lib = _native.load_library()
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/acch_b200.h but not exported"
    # the Python binding covers exactly the declared surface
    assert set(_native.SIGNATURES) == set(syms)
    assert lib.acch_abi_version() == 1


def test_stencil_offsets_table():
    from paper_2007_04560_b200 import _native
    import ctypes
    lib = _native.load_library()
    assert lib.acch_stencil_offsets(2, None) == 13
    assert lib.acch_stencil_offsets(3, None) == 25
    buf = (ctypes.c_int32 * 75)()
    n = lib.acch_stencil_offsets(3, buf)
    offs = {(buf[3 * i], buf[3 * i + 1], buf[3 * i + 2]) for i in range(n)}
    assert offs == {(x, y, z) for x in range(-2, 3) for y in range(-2, 3) for z in range(-2, 3)
                    if abs(x) + abs(y) + abs(z) <= 2}


def test_no_gpu_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2007_04560_b200.grid import BoundaryCondition, Grid
    from paper_2007_04560_b200.physics import State
    grid = Grid((4, 4), (1.0, 1.0), BoundaryCondition.PERIODIC)
    with pytest.raises(RuntimeError, match="CUDA"):
        State.from_interior(grid, np.full((4, 4), 0.5), np.zeros((4, 4)))


def test_partition_matches_reference_golden():
    from paper_2007_04560_b200.grid import BoundaryCondition, Grid
    from paper_2007_04560_b200.linalg import partition
    z = golden("partition.npz")
    for n in range(int(z["n_cases"])):
        meta = z[f"c{n}_meta"]
        dim = int(meta[6])
        counts = tuple(int(c) for c in meta[:dim])
        bc = BoundaryCondition.PERIODIC if meta[3] else BoundaryCondition.NEUMANN
        d = partition(Grid(counts, tuple(1.0 for _ in counts), bc), int(meta[4]), int(meta[5]))
        assert np.array_equal(np.concatenate(d.owned_cells), z[f"c{n}_owned"])
        assert np.array_equal([len(c) for c in d.extended_cells], z[f"c{n}_ext_len"])
        assert np.array_equal(np.concatenate(d.extended_cells), z[f"c{n}_ext"])
        assert np.array_equal(np.concatenate(d.owned_in_extended), z[f"c{n}_pos"])


def test_partition_errors():
    from paper_2007_04560_b200.exceptions import PartitionError
    from paper_2007_04560_b200.grid import BoundaryCondition, Grid
    from paper_2007_04560_b200.linalg import partition
    g = Grid((4, 4), (1.0, 1.0), BoundaryCondition.NEUMANN)
    with pytest.raises(PartitionError):
        partition(g, 0, 1)
    with pytest.raises(PartitionError):
        partition(g, 4, -1)
    with pytest.raises(PartitionError):
        partition(g, 17 * 19, 1)


def test_grid_and_params_validation():
    from paper_2007_04560_b200.grid import BoundaryCondition, Grid
    from paper_2007_04560_b200.physics import Params
    with pytest.raises(ValueError):
        Grid((3, 8), (1.0, 1.0), BoundaryCondition.NEUMANN)
    with pytest.raises(ValueError):
        Grid((8,), (1.0,), BoundaryCondition.NEUMANN)
    with pytest.raises(ValueError):
        Params(0.0, 1.0, 1.0, 1.0, 1.0)
    g = Grid((8, 6, 4), (1.0, 2.0, 3.0), BoundaryCondition.PERIODIC)
    assert g.array_shape == (4, 6, 8) and g.n_cells == 192 and g.dim == 3


# --- step controller: the reference's test_timestep.py cases, host path ----

def _ctl(**kw):
    from paper_2007_04560_b200.timestep import StepController
    base = dict(dt_min=1e-4, dt_max=10.0, eta=1e4)
    base.update(kw)
    return StepController(**base)


def test_controller_frozen_prediction():
    ctl = _ctl()
    assert ctl.predict_dt(np.full(4, 2.0), np.zeros(4), 2.0) == pytest.approx(0.09999500037496875, rel=1e-12)


def test_controller_limits_and_modes():
    ctl = _ctl()
    x = np.ones(8)
    assert ctl.predict_dt(x, x, 1.0) == 10.0
    assert ctl.predict_dt(x + 1e9, x, 1e-6) == 1e-4
    assert _ctl().initial_dt() == 1e-4
    assert _ctl(fixed_dt=0.5).initial_dt() == 0.5
    assert _ctl(fixed_dt=0.5).predict_dt(np.ones(2), np.zeros(2), 1.0) == 0.5


def test_controller_divergence_rules():
    from paper_2007_04560_b200.exceptions import SolverStallError
    ctl = _ctl()
    dt = ctl.on_divergence(1.0)
    assert dt == pytest.approx(1.0 / np.sqrt(2.0), rel=1e-14)
    assert ctl.eta == 2e4 and ctl.divergence_count == 1
    assert _ctl().on_divergence(1.2e-4) == 1e-4
    ctl = _ctl(max_retries_at_min=5)
    for _ in range(4):
        ctl.on_divergence(1e-4)
    with pytest.raises(SolverStallError):
        ctl.on_divergence(1e-4)
    ctl = _ctl(max_retries_at_min=3)
    ctl.on_divergence(1e-4)
    ctl.on_divergence(1e-4)
    ctl.note_success()
    ctl.on_divergence(1e-4)
    ctl.on_divergence(1e-4)
    with pytest.raises(SolverStallError):
        _ctl(fixed_dt=0.1).on_divergence(0.1)


def test_newton_config_and_solver_spec():
    from paper_2007_04560_b200.linalg import SubdomainSolverSpec
    from paper_2007_04560_b200.newton import NewtonConfig, should_refactor
    with pytest.raises(ValueError):
        NewtonConfig(rel_tol=0.0)
    with pytest.raises(ValueError):
        NewtonConfig(max_iterations=0)
    with pytest.raises(ValueError):
        NewtonConfig(backtrack_factor=1.5)
    assert should_refactor(0) and not should_refactor(3) and should_refactor(3, reuse_enabled=False)
    assert str(SubdomainSolverSpec.from_string("ILU2")) == "ilu2"
    assert SubdomainSolverSpec.from_string("lu").kind == "lu"
    with pytest.raises(ValueError):
        SubdomainSolverSpec.from_string("ilu")


def test_initial_fields_bitwise_reference_draw_order():
    from paper_2007_04560_b200.drivers import InitialSpec, RunConfig, TimeSpec, initial_fields
    from paper_2007_04560_b200.grid import BoundaryCondition, Grid
    from paper_2007_04560_b200.physics import Params
    from oracle import acch_oracle as O
    g = Grid((16, 8), (1.0, 1.0), BoundaryCondition.PERIODIC)
    cfg = RunConfig(g, Params(4.0, 2.0, 0.005, 0.1, 0.001), InitialSpec("random_uniform", 0.5, 0.05, 1234),
                    TimeSpec(1.0))
    u, v = initial_fields(cfg)
    uo, vo = O.initial_fields(O.Mesh((16, 8), (1.0, 1.0), True), 0.5, 0.05, 1234)
    assert np.array_equal(u, uo) and np.array_equal(v, vo)


def test_bench_arms_share_one_workload_config():
    """Both bench arms print the same `config` dict (the driver compares them)
    and the work-count table holds the windows the driver runs."""
    import importlib.util
    import json
    import sys
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    argv, sys.argv = sys.argv, ["bench.py", "--gpus", "1", "--steps", "20", "--warmup", "5"]
    try:
        spec.loader.exec_module(bench)
        args = bench.parse_args()
    finally:
        sys.argv = argv
    a = bench.workload_config(args)
    b = bench.workload_config(args, 1)
    assert a == b and a["workload"] == bench.workload_name(args)
    assert a["grid"] == [256, 256, 256] and a["subdomains"] == 32768
    assert "steps 6..25" in a["steps_timed"]
    counts, key = bench.load_counts(args)
    assert key == bench.window_key(args) and counts["gmres"] > 0
    table = json.load(open(os.path.join(ROOT, "bench_counts.json")))
    assert "256^3:box8:ilu0:ras-left:r30:W3:K4" in table
