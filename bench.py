#!/usr/bin/env python
"""Benchmark: adaptive NKS time steps of the AC/CH step on a synthetic
256^3 periodic grid (BASELINE.json configs[3]) through the library's public
API, plus the Jacobian-matvec and residual microbenchmarks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Prints ONE JSON line (rank 0).  `value` = accepted time steps per second over
exactly K timed steps after W warm-up steps (inputs resident in HBM); `e2e`
repeats K steps through the public API with the state staged from pinned host
memory and read back every step; `roofline` is for the kernel category with
the largest share of the timed region (algorithmic bytes / measured time,
from CUDA events recorded around every launch on the launching stream);
`cpu_baseline` times the unmodified reference package (baseline/_ref) by parts
on a bounded 32^3 sample on this host and composes a 256^3 step from the
window's work counts (see "CPU baseline / reference arm" below).  Every vector is 268 MB (> 126 MB L2), so no L2
flush is needed between iterations.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


METRIC = "NKS time steps/s (fp64, 256^3 adaptive); Jacobian-matvec GDOF/s; % of HBM roofline"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return dict(PEAKS_FALLBACK)


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=256, help="cells per axis (BASELINE configs[3]: 256)")
    ap.add_argument("--dim", type=int, default=3)
    ap.add_argument("--box", type=int, default=8, help="RAS box edge in cells")
    ap.add_argument("--solver", default="ilu0")
    ap.add_argument("--overlap", type=int, default=1)
    ap.add_argument("--variant", default="ras-left")
    ap.add_argument("--restart", type=int, default=30)
    ap.add_argument("--ortho", default="dcgs2", choices=["cgs2", "dcgs2", "mgs"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-micro", action="store_true", help="reference arm: skip the full-size microbenchmarks")
    ap.add_argument("--record-counts", action="store_true",
                    help="write this window's per-step work counts into bench_counts.json")
    ap.add_argument("--verbose", action="store_true")
    return ap.parse_args()


def log(args, *a):
    if args.verbose:
        print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        if not sm:
            return None
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# configuration
# ---------------------------------------------------------------------------

def make_config(args, world=1, rank=0):
    from paper_2007_04560_b200.drivers import InitialSpec, RunConfig, SolverSpec, TimeSpec
    from paper_2007_04560_b200.grid import BoundaryCondition, Grid
    from paper_2007_04560_b200.linalg import SchwarzVariant, SubdomainSolverSpec
    from paper_2007_04560_b200.physics import Params
    n = args.n
    counts = (n,) * args.dim
    grid = Grid(counts, (1.0,) * args.dim, BoundaryCondition.PERIODIC)
    if world > 1:
        # z-slab decomposition: this rank's planes, halos + reductions over NCCL
        from paper_2007_04560_b200.slab import NcclComm, bind_comm, split_grid
        grid = split_grid(grid, world, rank)
        bind_comm(grid, NcclComm(periodic=True))     # in-library NCCL halos + allreduces on the solver stream
    nsub = (n // args.box) ** args.dim
    cfg = RunConfig(grid, Params(4.0, 2.0, 0.005, 0.1, 0.001),
                    InitialSpec("random_uniform", 0.5, 0.01, 1234),
                    TimeSpec(horizon=10.0, mode="adaptive", dt_min=1e-4, dt_max=10.0),
                    SolverSpec(preconditioner=SchwarzVariant(args.variant), overlap=args.overlap,
                               subdomain_solver=SubdomainSolverSpec.from_string(args.solver), subdomains=nsub,
                               gmres_restart=args.restart, orthogonalization=args.ortho))
    return cfg, nsub


def workload_config(args, world=None):
    """The workload both arms are quoted on (identical dict in both JSON lines)."""
    world = args.gpus if world is None else world
    nsub = (args.n // args.box) ** args.dim
    vec_mb = 16 * args.n ** args.dim / 1e6
    return {"workload": workload_name(args), "grid": [args.n] * args.dim, "bc": "periodic",
            "ic": "u0=0.5+0.01U(-1,1), v0=0.01U(-1,1), seed 1234", "subdomains": nsub,
            "parallelism": "1 GPU" if world == 1 else
            f"z-slabs over {world} GPUs (2 ghost planes; in-library NCCL halos + allreduces)",
            "l2": f"every vector {vec_mb:.0f} MB vs 126 MB L2" + (" (no flush needed)" if vec_mb > 126 else ""),
            "steps_timed": f"accepted steps {args.warmup + 1}..{args.warmup + args.steps} "
                           f"(after {args.warmup} warm-up steps)"}


def workload_name(args):
    return (f"AC/CH {args.dim}D {args.n}^{args.dim} periodic fp64, adaptive dt (eta=1e2), NKS: Newton + "
            f"GMRES({args.restart}) + {args.variant} {args.box}^{args.dim}-cell boxes overlap {args.overlap} {args.solver}")


# ---------------------------------------------------------------------------
# CPU baseline / reference arm: the UNMODIFIED reference package `acch`
# ---------------------------------------------------------------------------
#
# The reference (pure Python + numpy / scipy / numba) is installed, unmodified,
# into baseline/_ref (git-ignored; it travels to the GPU box with the repo):
#   python -m pip install --no-index --no-build-isolation --no-deps \
#       --target baseline/_ref <copy of /root/reference/pkg>
# It cannot run a 256^3 step on a host in useful time (its Jacobian assembly
# alone needs 47.7 GB and 242 s; one GMRES iteration ~17 s), so a step is
# timed by parts on a bounded sample: the same solver (left-RAS, 8^3-cell
# boxes, overlap 1, ILU(0), GMRES(30)) on a 32^3 periodic grid with the same
# seeded fields, each part timed with the reference's own functions --
# residual_vector, assemble_jacobian, SchwarzPreconditioner.update (numba
# ILU), one 30-iteration gmres cycle -- and composed into a 256^3 step with
# the cell ratio (every part is linear in the cell count) and the work counts
# of the timed window (GMRES iterations, Newton iterations, factorisations,
# residual evaluations), which bench_counts.json records per (warmup, steps)
# window from the GPU arm's own run of the identical workload; the GPU arm
# checks its counts against that table on every run.

REF_DIR = os.path.join(ROOT, "baseline", "_ref")
COUNTS_FILE = os.path.join(ROOT, "bench_counts.json")


def import_reference():
    """The reference package from baseline/_ref, or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "acch")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "acch_ref_numba"))
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import acch  # noqa: F401
        import acch.linalg  # noqa: F401
        return acch
    except Exception:
        return None


def window_key(args):
    ov = "" if args.overlap == 1 else f"ov{args.overlap}:"
    return f"{args.n}^{args.dim}:box{args.box}:{ov}{args.solver}:{args.variant}:r{args.restart}:W{args.warmup}:K{args.steps}"


def load_counts(args):
    """Per-step work of the timed window, recorded from the GPU arm."""
    try:
        table = json.load(open(COUNTS_FILE))
    except Exception:
        return None, None
    key = window_key(args)
    if key in table:
        return table[key], key
    # same workload, another window: nearest recorded window (stated in `sample`)
    pre = key.rsplit(":W", 1)[0] + ":W"
    cands = [k for k in table if k.startswith(pre)]
    if not cands:
        return None, None
    return table[cands[0]], cands[0]


def reference_parts(args, threads, ns=32, reps=1):
    """Seconds per call of each part of the reference's NKS step on an ns^dim
    sample (after a warm-up that compiles the numba ILU kernels)."""
    import numpy as np
    acch = import_reference()
    if acch is None:
        return None
    from acch.grid import BoundaryCondition as RBC, Field as RField, Grid as RGrid
    from acch.linalg import (SchwarzPreconditioner as RSP, SchwarzVariant as RSV, SubdomainSolverSpec as RSS,
                             gmres as rgmres, partition as rpartition)
    from acch.parallel import WorkerPool
    from acch.physics import Params as RParams, State as RState
    from acch.scheme import (StepProblem as RStep, assemble_jacobian as rjac, residual_vector as rres,
                             state_from_vector, vector_from_state)
    g = RGrid((ns,) * args.dim, (1.0,) * args.dim, RBC.PERIODIC)
    rng = np.random.default_rng(1234)
    u = 0.5 + rng.uniform(-0.01, 0.01, g.array_shape)
    v = rng.uniform(-0.01, 0.01, g.array_shape)
    old = RState(RField.from_interior(g, u), RField.from_interior(g, v))
    prob = RStep.create(g, RParams(4.0, 2.0, 0.005, 0.1, 0.001), old, 0.0111)
    x = vector_from_state(old) + 1e-4 * np.random.default_rng(1234).standard_normal(2 * g.n_cells)
    new = state_from_vector(g, x)
    nsub = (ns // args.box) ** args.dim
    out = {}
    with WorkerPool(threads) as pool:
        pre = RSP(rpartition(g, nsub, 1), RSV(args.variant), RSS.from_string(args.solver), pool)
        F = rres(prob, new)
        J = rjac(prob, new)
        pre.update(J)                                        # numba compile (factor)
        rgmres(J.matvec, -F, pre, 1e-30, 1e-300, 2, 2)       # numba compile (solve)
        ts = {"residual": [], "jacobian": [], "factor": [], "gmres_iter": []}
        for _ in range(reps):
            t0 = time.perf_counter(); F = rres(prob, new); ts["residual"].append(time.perf_counter() - t0)
            t0 = time.perf_counter(); J = rjac(prob, new); ts["jacobian"].append(time.perf_counter() - t0)
            pre.invalidate()
            t0 = time.perf_counter(); pre.update(J); ts["factor"].append(time.perf_counter() - t0)
            t0 = time.perf_counter()
            res = rgmres(J.matvec, -F, pre, 1e-30, 1e-300, args.restart, args.restart)   # exactly one cycle
            ts["gmres_iter"].append((time.perf_counter() - t0) / max(res.iterations, 1))
        for k, vals in ts.items():
            out[k] = min(vals)
    out["cells"] = g.n_cells
    out["ns"] = ns
    return out


def reference_step_estimate(args, parts, counts):
    scale = float(args.n ** args.dim) / parts["cells"]
    t = scale * (counts["gmres"] * parts["gmres_iter"] + counts["factorizations"] * parts["factor"] +
                 counts["jacobians"] * parts["jacobian"] + counts["residuals"] * parts["residual"])
    return t, scale


def reference_microbench(args, threads):
    """the unmodified residual_vector at the bench grid
    and StencilMatrix.matvec at 128^3 (assembly at 256^3 needs 47.7 GB), on
    the microbenchmark state pair U' = U^n + 1e-4 N(0,1)."""
    import numpy as np
    if import_reference() is None:
        return None
    from acch.grid import BoundaryCondition as RBC, Field as RField, Grid as RGrid
    from acch.physics import Params as RParams, State as RState
    from acch.scheme import (StepProblem as RStep, assemble_jacobian as rjac, residual_vector as rres,
                             state_from_vector, vector_from_state)
    out = {}
    for name, n in (("residual", args.n), ("matvec", min(args.n, 128))):
        g = RGrid((n,) * args.dim, (1.0,) * args.dim, RBC.PERIODIC)
        rng = np.random.default_rng(1234)
        u = 0.5 + rng.uniform(-0.01, 0.01, g.array_shape)
        v = rng.uniform(-0.01, 0.01, g.array_shape)
        old = RState(RField.from_interior(g, u), RField.from_interior(g, v))
        prob = RStep.create(g, RParams(4.0, 2.0, 0.005, 0.1, 0.001), old, 1e-4)
        x = vector_from_state(old) + 1e-4 * np.random.default_rng(1234).standard_normal(2 * g.n_cells)
        new = state_from_vector(g, x)
        if name == "residual":
            t0 = time.perf_counter()
            rres(prob, new)
            t = time.perf_counter() - t0
        else:
            t0 = time.perf_counter()
            J = rjac(prob, new)
            t_asm = time.perf_counter() - t0
            w = np.random.default_rng(7).standard_normal(2 * g.n_cells)
            ts = []
            for _ in range(3):
                t0 = time.perf_counter()
                J.matvec(w)
                ts.append(time.perf_counter() - t0)
            t = min(ts)
            out["matvec_assembly_s"] = t_asm
        out[name] = {"grid": [n] * args.dim, "s": t, "gdof_s": 2 * g.n_cells / t / 1e9}
        del prob, new, old
    out["config1"] = reference_config1(threads)
    out["threads"] = threads
    out["kind"] = "reference"
    return out


def reference_config1(threads):
    """BASELINE configs[0] (64^2 periodic, 10 fixed steps
    of 1e-4, left-RAS 2x2, overlap 1, ILU(0)) run in full through the
    unmodified reference's `simulate` (cli/drivers.py:76-184) at 1 and T host
    threads, after one warm-up run (numba compilation)."""
    try:
        from acch.cli.config import InitialSpec as RI, RunConfig as RC, SolverSpec as RS, TimeSpec as RT
        from acch.cli.drivers import simulate as rsim
        from acch.grid import BoundaryCondition as RBC, Grid as RGrid
        from acch.linalg import SchwarzVariant as RV, SubdomainSolverSpec as RSub
        from acch.physics import Params as RParams
        cfg = RC(RGrid((64, 64), (1.0, 1.0), RBC.PERIODIC), RParams(4.0, 2.0, 0.005, 0.1, 0.001),
                 RI("random_uniform", 0.5, 0.05, 1234), RT(horizon=1e-3, mode="fixed", dt=1e-4),
                 RS(RV.LEFT_RAS, 1, RSub("ilu", 0), subdomains=4))
        rsim(cfg, threads=1, max_steps=2)
        out = {}
        for th in sorted({1, min(threads, 4)}):
            t0 = time.perf_counter()
            res = rsim(cfg, threads=th, max_steps=10)
            t = time.perf_counter() - t0
            rows = res.history
            out[f"threads_{th}"] = {"steps": len(rows) - 1, "s": t, "steps_s": (len(rows) - 1) / t,
                                    "energy_last": rows[-1].energy}
        return out
    except Exception as e:      # reported, never fatal for the arm
        return {"error": f"{type(e).__name__}: {e}"}


def cpu_sample(args, threads=1, counts=None, ns=None):
    """The reference's step cost on this host (see above); falls back to the
    oracle port (numpy + C ILU, tests only) when the reference package is not
    importable."""
    counts = counts or load_counts(args)[0]
    parts = reference_parts(args, threads, ns or 32) if import_reference() is not None else None
    if parts is not None and counts is not None:
        t_step, scale = reference_step_estimate(args, parts, counts)
        return {"value": 1.0 / t_step, "unit": "time steps/s", "cores": threads, "kind": "reference",
                "parts_s": {k: parts[k] for k in ("residual", "jacobian", "factor", "gmres_iter")},
                "sample": (f"unmodified reference acch (baseline/_ref) on {parts['ns']}^{args.dim} periodic, "
                           f"{args.box}^{args.dim}-cell boxes, {args.solver}, {threads} thread(s): "
                           f"{parts['gmres_iter'] * 1e3:.1f} ms per GMRES iteration, {parts['factor']:.3f} s per "
                           f"factorisation, {parts['jacobian']:.3f} s per assembly, {parts['residual'] * 1e3:.1f} ms "
                           f"per residual; x{scale:.0f} cells, per-step counts {counts['gmres']:.1f} GMRES + "
                           f"{counts['factorizations']:.2f} factorisations + {counts['jacobians']:.2f} Jacobians + "
                           f"{counts['residuals']:.2f} residuals (bench_counts.json); step estimate {t_step:.0f} s")}
    # fallback: the oracle port
    import numpy as np
    from oracle import acch_oracle as O
    if counts is None:
        return {"error": "no recorded per-step counts for this workload (bench_counts.json)"}
    ns = ns or 32
    m = O.Mesh((ns,) * args.dim, (1.0,) * args.dim, True)
    u, v = O.initial_fields(m, 0.5, 0.01, 1234)
    st = O.Step(m, O.Coeffs(), u, v, 2e-3)
    x = O.pack(u, v) + 1e-4 * np.random.default_rng(1234).standard_normal(2 * m.n_cells)
    pre = O.SchwarzOracle(O.decompose(m, (ns // args.box) ** args.dim, 1), args.variant, args.solver, threads)
    t0 = time.perf_counter()
    J = st.jacobian(x)
    pre.update(J.assemble_fast())
    t_fact = time.perf_counter() - t0
    b = -st.residual(x)
    t0 = time.perf_counter()
    res = O.gmres(J.matvec, b, pre.apply, 1e-30, 1e-300, args.restart, args.restart)
    t_gm = (time.perf_counter() - t0) / max(res.iterations, 1)
    scale = float(args.n ** args.dim) / m.n_cells
    t_step = scale * (counts["gmres"] * t_gm + counts["factorizations"] * t_fact)
    return {"value": 1.0 / t_step, "unit": "time steps/s", "cores": threads, "kind": "port",
            "sample": (f"oracle port (reference not importable) on {ns}^{args.dim}: {t_gm * 1e3:.1f} ms per GMRES "
                       f"iteration, {t_fact:.2f} s per assembly+factorisation, x{scale:.0f} cells, "
                       f"{counts['gmres']:.1f} GMRES + {counts['factorizations']:.2f} factorisations per step")}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    counts, key = load_counts(args)
    vals, sample = [], None
    micro = None
    t_start = time.perf_counter()
    for i in range(min(args.warmup, 1) + args.steps):
        r = cpu_sample(args, threads=threads, counts=counts)
        if "value" not in r:
            print(json.dumps({"impl": "reference", "unavailable": r.get("error", "no sample")}), flush=True)
            return
        if i >= min(args.warmup, 1):
            vals.append(r["value"])
            sample = r
        if i == 0 and r["kind"] == "reference" and not args.no_micro:
            micro = reference_microbench(args, threads)
    value = sum(vals) / len(vals)
    line = {"metric": METRIC, "value": value, "unit": "time steps/s",
            "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args),
            "arm": {"runs_on": f"host CPU, {threads} threads (the reference's WorkerPool)", "counts_window": key},
            "cpu_baseline": {"value": value, "unit": "time steps/s", "cores": threads, "kind": sample["kind"],
                             "sample": sample["sample"], "parts_s": sample.get("parts_s")},
            "reference_microbench": micro,
            "e2e": {"value": value, "unit": "time steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": time.perf_counter() - t_start}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def measured_traffic(category):
    """DRAM bytes (read + write) per launch of the dominant kernel category
    from the committed `ncu --set full` captures (profiles/traffic.json,
    written by tools/ncu_traffic.py); None when not captured."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if category not in ("precond_apply", "matvec") or not os.path.exists(path):
        return None, None
    ent = [v for v in json.load(open(path)).values() if v.get("category") == category]
    if not ent:
        return None, None
    return sum(v["traffic_bytes"] for v in ent), "ncu --set full: " + ", ".join(v["source"] for v in ent)


def measured_issue(category):
    """Instruction-issue evidence for a compute-heavy kernel from the committed
    `ncu --set full` capture (profiles/traffic.json): warp instructions per
    launch, FP64-pipe and issue-slot utilisation.  The residual is bound by
    FP64 issue, not HBM, so its roofline is stated in both."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(path):
        return None
    ent = [v for v in json.load(open(path)).values() if v.get("category") == category and "inst_executed" in v]
    if not ent:
        return None
    e = ent[0]
    return {"warp_inst_per_launch": e["inst_executed"], "fp64_pipe_pct": e.get("fp64_pipe_pct"),
            "issue_active_pct": e.get("issue_active_pct"), "source": "ncu --set full: " + e["source"]}


def microbench_stencils(args, stepper, peaks, reps=20):
    """Standalone residual and Jacobian-matvec launches at the current state
    (U' = U^n + 1e-4 N(0,1): the chords take the series branch)."""
    import torch
    from paper_2007_04560_b200.physics import State
    from paper_2007_04560_b200.scheme import StepProblem, assemble_jacobian
    grid = stepper.grid
    n2 = 2 * grid.n_cells
    prob = StepProblem.create(grid, stepper.config.params, stepper.state, 1e-4)
    gen = torch.Generator(device=stepper.state.device).manual_seed(1234)
    pert = stepper.state.vector + 1e-4 * torch.randn(n2, dtype=torch.float64, device=stepper.state.device,
                                                     generator=gen)
    new = State(grid, pert)
    J = assemble_jacobian(prob, new)
    w = torch.randn(n2, dtype=torch.float64, device=pert.device, generator=gen)
    y = torch.empty_like(w)
    F = torch.empty_like(w)
    out = {}
    for name, fn, nbytes in (("matvec", lambda: J.matvec_into(w, y), 88.0 * grid.n_cells),
                             ("residual", lambda: prob.residual_into(pert, F), 48.0 * grid.n_cells)):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(reps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            fn() if name == "matvec" else _residual_async(prob, pert, F)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        t = ts[len(ts) // 2] * 1e-3
        gbs = nbytes / t / 1e9
        out[name] = {"ms": t * 1e3, "gdof_s": n2 / t / 1e9, "gb_s": gbs, "frac": gbs / peaks["hbm_gbs"],
                     "alg_bytes": nbytes}
        iss = measured_issue(name)
        if iss is not None:
            # issue roofline: 148 SMs x 4 schedulers x 1 warp instruction per clock
            clk = float(os.environ.get("ACCH_SM_MHZ", "1965")) * 1e6
            t_issue = iss["warp_inst_per_launch"] / (148 * 4 * clk)
            iss.update({"issue_bound_ms": t_issue * 1e3, "issue_frac": t_issue / t, "clock_mhz_assumed": clk / 1e6})
            out[name]["issue"] = iss
    return out


def _residual_async(prob, x, F):
    # the public residual synchronises to return ||F|| and the gap; for the
    # launch-time microbenchmark call the kernel without the readback
    from paper_2007_04560_b200 import _native as nat
    import ctypes
    nat.check(nat.lib().acch_residual(prob.ctx.bind(), nat.ptr(prob.old.x), prob.dt, nat.ptr(x), nat.ptr(F),
                                      None, None), "residual")


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2007_04560_b200 import _native as nat
    from paper_2007_04560_b200.drivers import Stepper, build_initial_state
    from paper_2007_04560_b200.physics import State

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    peaks = load_peaks()
    cfg, nsub = make_config(args, world, rank)
    grid = cfg.grid
    t_setup = time.perf_counter()
    state = build_initial_state(cfg, device=dev)
    stepper = Stepper(cfg, state)
    ctx = nat.context_for(grid, cfg.params, dev)
    log(args, f"setup {time.perf_counter() - t_setup:.1f}s")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for i in range(args.warmup):
        t0 = time.perf_counter()
        dt, nn, ng = stepper.advance()
        torch.cuda.synchronize()
        log(args, f"warmup step {stepper.step}: dt={dt:.4g} newton={nn} gmres={ng} "
                  f"retries={len(stepper.events)} {time.perf_counter() - t0:.2f}s")

    first_timed = stepper.step + 1
    snap = stepper.snapshot()      # the e2e pass replays exactly these K steps
    ctx.profile(True)
    ctx.profile_read()
    launches0 = nat.total_launches()
    comm0 = ctx.comm_stats()
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    newton_total = gmres_total = 0
    ev_before = len(stepper.events)
    dts = []
    for i in range(args.steps):
        t0 = time.perf_counter()
        dt, nn, ng = stepper.advance()
        newton_total += nn
        gmres_total += ng
        dts.append(dt)
        log(args, f"timed step {stepper.step}: dt={dt:.4g} newton={nn} gmres={ng} "
                  f"retries={len(stepper.events)} {time.perf_counter() - t0:.2f}s")
    e1.record()
    barrier()
    elapsed = e0.elapsed_time(e1) * 1e-3
    clk = clocks.stop()
    prof = ctx.profile_read()
    ctx.profile(False)
    comm1 = ctx.comm_stats()
    comm = {"halo_bytes_per_step": (comm1["halo_bytes"] - comm0["halo_bytes"]) / max(args.steps, 1),
            "nccl_calls_per_step": (comm1["nccl_calls"] - comm0["nccl_calls"]) / max(args.steps, 1),
            "data_plane": "in-library NCCL (send/recv ghost planes, allreduce) on the solver stream"} \
        if world > 1 else None
    launches = nat.total_launches() - launches0
    if world > 1:
        t = torch.tensor([elapsed], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    retries = len(stepper.events) - ev_before

    # e2e: the same K steps again (replayed from the snapshot) through the
    # public API, with the state staged from pinned host memory each step
    e2e = None
    n2 = 2 * grid.n_cells
    if not args.no_e2e:
        host = torch.empty((grid.n_store, 2), dtype=torch.float64, pin_memory=True)
        stepper.restore(snap)
        host.copy_(stepper.state.x)
        barrier()
        t0 = time.perf_counter()
        e2e_gmres = 0
        for i in range(args.steps):
            dev_state = State(grid, host.to(dev, non_blocking=True))
            stepper.state = dev_state
            stepper.x_now = dev_state.vector
            e2e_gmres += stepper.advance()[2]
            host.copy_(stepper.state.x, non_blocking=True)
            torch.cuda.synchronize()
        barrier()
        t_e2e = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([t_e2e], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            t_e2e = float(t.item())
        e2e = {"value": args.steps / t_e2e, "unit": "time steps/s", "h2d_bytes_per_step": 16 * grid.n_store,
               "d2h_bytes_per_step": 16 * grid.n_store, "gmres": e2e_gmres,
               "note": "the timed K steps replayed from a snapshot (same work as `value`)"}

    micro = microbench_stencils(args, stepper, peaks)

    total_ms = sum(v[0] for v in prof.values())
    cats = {}
    for k, (ms, cnt, nb) in prof.items():
        if cnt == 0:
            continue
        gbs = nb / (ms * 1e-3) / 1e9 if ms > 0 else 0.0
        cats[k] = {"ms": round(ms, 3), "share": round(ms / (elapsed * 1e3), 4), "launches": int(cnt),
                   "alg_bytes_per_launch": nb / cnt, "gb_s": round(gbs, 1),
                   "frac": round(gbs / peaks["hbm_gbs"], 4)}
    dom = max(cats, key=lambda k: cats[k]["ms"]) if cats else "matvec"
    d = cats.get(dom, {})
    traffic, traffic_src = measured_traffic(dom)
    roofline = {"bound": "hbm", "kernel": dom, "achieved": d.get("gb_s"), "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": d.get("frac"), "traffic": traffic, "traffic_source": traffic_src,
                "avg_launch_ms": (d["ms"] / d["launches"]) if d else None,
                "alg_bytes_per_launch": d.get("alg_bytes_per_launch"), "peak_source": peaks["source"]}

    # per-step work of the timed window (the reference arm composes its step
    # from these; bench_counts.json pins them per window)
    steps_done = max(args.steps, 1)
    counts = {"gmres": gmres_total / steps_done, "newton": newton_total / steps_done,
              "factorizations": prof.get("precond_factor", (0, 0, 0))[1] / steps_done,
              "jacobians": prof.get("jacobian_prepare", (0, 0, 0))[1] / steps_done,
              "residuals": prof.get("residual", (0, 0, 0))[1] / steps_done, "retries": retries / steps_done}
    counts_check = None
    if world == 1:
        rec, key = load_counts(args)
        if args.record_counts and rank == 0:
            try:
                table = json.load(open(COUNTS_FILE))
            except Exception:
                table = {}
            table[window_key(args)] = counts
            with open(COUNTS_FILE, "w") as f:
                json.dump(table, f, indent=1, sort_keys=True)
            counts_check = "recorded"
        elif rec is not None and key == window_key(args):
            bad = {k: (counts[k], rec.get(k)) for k in ("gmres", "newton", "factorizations", "jacobians", "residuals")
                   if rec.get(k) is None or abs(counts[k] - rec[k]) > 1e-9 * max(1.0, abs(rec[k]))}
            counts_check = "match" if not bad else {"MISMATCH": bad}
            if bad and rank == 0:
                print(f"bench.py: WARNING: the timed window's work counts differ from bench_counts.json[{key}]: "
                      f"{bad} -- the reference arm's step estimate is keyed to the recorded counts", file=sys.stderr,
                      flush=True)
        else:
            counts_check = "no recorded counts for this window"

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_sample(args, threads=1, counts=counts)
        except Exception as e:  # the baseline must not break the GPU line
            cpu = {"error": repr(e)}

    if rank == 0:
        value = args.steps / elapsed
        line = {
            "metric": METRIC,
            "value": value, "unit": "time steps/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": elapsed * 1e3 / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, world),
            "solver_stats": {"newton": newton_total, "gmres": gmres_total, "retries": retries,
                             "dt": [round(x, 6) for x in dts], "per_step": counts, "counts_check": counts_check,
                             "ms_per_gmres_iteration": elapsed * 1e3 / max(gmres_total, 1)},
            "roofline": roofline,
            "matvec": micro["matvec"], "residual": micro["residual"],
            "kernels": cats,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "comm": comm,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
