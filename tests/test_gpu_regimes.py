"""Multi-step histories at the BASELINE solver regimes, against the
unmodified reference (tests/golden/make_golden.py `sim3p`, `sim2a`, `sim4a`):

* c3proxy  -- config 3's stiffness (dx = 1/128) on 32^3 Neumann cells in a box
              of side 0.25, 8^3-cell boxes, ILU(2) (ILU(0)/ILU(1) fail there),
              eta = 1e2, 3 adaptive steps;
* c2analog -- config 2's solver on 128^2 periodic: 16x16-cell boxes, exact LU,
              eta = 1e4, 20 adaptive steps with divergence retries;
* c4analog -- the bench's regime on 32^3 periodic: 8^3-cell boxes, ILU(0),
              eta = 1e2, 5 adaptive steps with divergence retries.

Each runs on the production defaults (lagged CGS2 with the device-resident
Arnoldi loop, the class-group / warp-wide Schwarz solvers) and on the
reference-order classical Gram-Schmidt.  Pass: the same accepted-dt sequence
(1e-10), the same Newton counts and divergence events, GMRES within +-2 per
step, fields <= 1e-8 relative L2, monotone energy, mass at round-off."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

from paper_2007_04560_b200.grid import BoundaryCondition, Grid  # noqa: E402
from paper_2007_04560_b200.linalg import SchwarzVariant, SubdomainSolverSpec  # noqa: E402
from paper_2007_04560_b200.physics import Params  # noqa: E402

PARAMS = Params(4.0, 2.0, 0.005, 0.1, 0.001)
DEV = "cuda:0"


def run(tag, ortho):
    from paper_2007_04560_b200.drivers import InitialSpec, RunConfig, SolverSpec, TimeSpec, simulate
    z = golden(f"sim_{tag}.npz")
    counts = tuple(int(c) for c in z["counts"])
    L = float(z["length"])
    bc = BoundaryCondition.PERIODIC if bool(z["periodic"]) else BoundaryCondition.NEUMANN
    g = Grid(counts, tuple(L for _ in counts), bc)
    center, amp, dt, horizon, nsub, eta, max_steps = (float(t) for t in z["meta"])
    cfg = RunConfig(g, PARAMS, InitialSpec("random_uniform", center, amp, 1234),
                    TimeSpec(horizon=horizon, mode=str(z["mode"]), dt=dt, dt_min=1e-4, dt_max=10.0,
                             eta=None if eta < 0 else eta),
                    SolverSpec(preconditioner=SchwarzVariant(str(z["variant"])),
                               subdomain_solver=SubdomainSolverSpec.from_string(str(z["solver"])),
                               subdomains=int(nsub), orthogonalization=ortho))
    assert cfg.eta == float(z["eta"])
    res = simulate(cfg, max_steps=None if max_steps < 0 else int(max_steps), device=DEV)
    return z, res


def check(z, res):
    ref = z["rows"]
    assert res.status == str(z["status"])
    got = np.array([[r.step, r.time, r.dt, r.energy, r.mass_u, r.max_abs_v, r.newton, r.gmres]
                    for r in res.history])
    assert got.shape == ref.shape
    assert res.controller.divergence_count == int(z["divergences"])
    np.testing.assert_allclose(got[:, 2], ref[:, 2], rtol=1e-10)   # accepted dt sequence
    np.testing.assert_array_equal(got[:, 6], ref[:, 6])            # Newton iterations
    assert np.all(np.abs(got[:, 7] - ref[:, 7]) <= 2), (got[:, 7], ref[:, 7])
    np.testing.assert_allclose(got[:, 3], ref[:, 3], rtol=1e-10)   # energy
    np.testing.assert_allclose(got[:, 4], ref[:, 4], rtol=1e-12)   # mass
    u, v = res.final_state.to_numpy()
    err = np.sqrt(np.sum((u - z["u"]) ** 2 + (v - z["v"]) ** 2) / np.sum(z["u"] ** 2 + z["v"] ** 2))
    assert err <= 1e-8, err
    e = got[:, 3]
    assert np.all(np.diff(e) <= 1e-8 * np.maximum(1.0, np.abs(e[1:])))
    ref_drift = np.max(np.abs(ref[:, 4] - ref[0, 4]))
    assert np.max(np.abs(got[:, 4] - got[0, 4])) <= max(2.0 * ref_drift, 1e-12)


@pytest.mark.parametrize("ortho", ["dcgs2", "cgs2"])
@pytest.mark.parametrize("tag", ["c3proxy", "c2analog", "c4analog"])
def test_baseline_regime_history_matches_reference(tag, ortho):
    check(*run(tag, ortho))
