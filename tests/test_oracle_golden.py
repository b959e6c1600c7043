"""Pin the CPU oracle against the reference's own outputs (tests/golden/*.npz).

These run on CPU only (no GPU, no /root/reference): the fixtures were produced
by tests/golden/make_golden.py from the unmodified reference package.
"""

import numpy as np
import pytest

from conftest import golden
from oracle import acch_oracle as O

CO = O.Coeffs()
STENCIL = ["2d_neu", "2d_per", "2d_per4", "3d_neu", "3d_per", "2d_per_big", "3d_neu_big"]


def mesh_of(z):
    counts = tuple(int(c) for c in z["counts"])
    return O.Mesh(counts, tuple(1.0 for _ in counts), bool(z["periodic"]))


def test_chord_battery_matches_reference():
    z = golden("chord.npz")
    val, der = O.chord(z["a"], z["b"], 10, want_deriv=True)
    # same branch predicates and formulas: agreement to a few ulps
    np.testing.assert_allclose(val, z["val"], rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(der, z["der"], rtol=1e-12, atol=1e-13)


def test_chord_known_answers():
    # physics golden values of the reference tests (test_physics.py:246-252)
    assert O.chord(0.6, 0.4) == 0.0
    assert abs(float(O.chord(0.7, 0.5)) - 0.41141439252525923) <= 1e-12


def test_local_energy_known_answer():
    # test_physics.py:82-86
    e = O.local_energy(CO, np.array(0.5), np.array(0.0), 0.0, 0.0)
    assert abs(float(e) - 0.36137056388801094) <= 1e-15


@pytest.mark.parametrize("tag", STENCIL)
def test_residual_matches_reference(tag):
    z = golden(f"stencil_{tag}.npz")
    m = mesh_of(z)
    st = O.Step(m, CO, z["uo"], z["vo"], float(z["dt"]))
    F = st.residual(O.pack(z["un"], z["vn"]))
    scale = np.max(np.abs(z["F"]))
    assert np.max(np.abs(F - z["F"])) <= 1e-12 * scale
    F0 = st.residual(O.pack(z["uo"], z["vo"]))
    assert np.max(np.abs(F0 - z["F0"])) <= 1e-12 * np.max(np.abs(z["F0"]))


@pytest.mark.parametrize("tag", STENCIL)
def test_jacobian_matvec_matches_reference(tag):
    z = golden(f"stencil_{tag}.npz")
    m = mesh_of(z)
    st = O.Step(m, CO, z["uo"], z["vo"], float(z["dt"]))
    J = st.jacobian(O.pack(z["un"], z["vn"]))
    y = J.matvec(z["w"])
    assert np.max(np.abs(y - z["Jw"])) <= 1e-12 * np.max(np.abs(z["Jw"]))


@pytest.mark.parametrize("tag", ["2d_neu", "2d_per", "2d_per4", "3d_neu", "3d_per"])
def test_assembled_blocks_match_reference(tag):
    z = golden(f"stencil_{tag}.npz")
    m = mesh_of(z)
    st = O.Step(m, CO, z["uo"], z["vo"], float(z["dt"]))
    ip, ix, bl = st.jacobian(O.pack(z["un"], z["vn"])).assemble()
    assert np.array_equal(ip, z["J_indptr"])
    assert np.array_equal(ix, z["J_indices"])
    scale = np.max(np.abs(z["J_blocks"]))
    assert np.max(np.abs(bl - z["J_blocks"])) <= 1e-12 * scale


@pytest.mark.parametrize("tag", STENCIL)
def test_energy_and_gap_match_reference(tag):
    z = golden(f"stencil_{tag}.npz")
    m = mesh_of(z)
    e = O.total_energy(m, CO, z["un"], z["vn"])
    assert abs(e - float(z["energy_new"])) <= 1e-13 * abs(float(z["energy_new"]))
    assert O.admissibility_gap(z["un"], z["vn"]) == float(z["gap"])


def test_partition_matches_reference():
    z = golden("partition.npz")
    for n in range(int(z["n_cases"])):
        meta = z[f"c{n}_meta"]
        dim = int(meta[6])
        counts = tuple(int(c) for c in meta[:dim])
        m = O.Mesh(counts, tuple(1.0 for _ in counts), bool(meta[3]))
        b = O.decompose(m, int(meta[4]), int(meta[5]))
        assert np.array_equal(np.concatenate(b.owned), z[f"c{n}_owned"])
        assert np.array_equal([len(c) for c in b.owned], z[f"c{n}_owned_len"])
        assert np.array_equal(np.concatenate(b.extended), z[f"c{n}_ext"])
        assert np.array_equal([len(c) for c in b.extended], z[f"c{n}_ext_len"])
        assert np.array_equal(np.concatenate(b.owned_pos), z[f"c{n}_pos"])


@pytest.mark.parametrize("tag", ["2d_neu", "2d_per", "3d_per", "3d_neu"])
@pytest.mark.parametrize("variant", ["asm", "ras-left", "ras-right"])
@pytest.mark.parametrize("solver", ["ilu0", "ilu1", "ilu2", "lu"])
def test_schwarz_apply_matches_reference(tag, variant, solver):
    z = golden(f"schwarz_{tag}.npz")
    m = mesh_of(z)
    st = O.Step(m, CO, z["uo"], z["vo"], float(z["dt"]))
    blocks = st.jacobian(O.pack(z["un"], z["vn"])).assemble()
    pre = O.SchwarzOracle(O.decompose(m, int(z["nsub"]), int(z["overlap"])), variant, solver)
    pre.update(blocks)
    out = pre.apply(z["r"])
    ref = z[f"{variant}_{solver}"]
    assert np.max(np.abs(out - ref)) <= 1e-10 * np.max(np.abs(ref))


def _gmres_setup():
    z = golden("gmres.npz")
    m = O.Mesh((16, 12), (1.0, 1.0), True)
    st = O.Step(m, CO, z["uo"], z["vo"], 1e-3)
    J = st.jacobian(O.pack(z["un"], z["vn"]))
    pre = O.SchwarzOracle(O.decompose(m, 4, 1), "ras-left", "ilu0")
    pre.update(J.assemble())
    return z, J, pre


def test_gmres_matches_reference():
    z, J, pre = _gmres_setup()
    b = z["b"]
    res = O.gmres(J.matvec, b, pre.apply, 1e-8, 1e-14, 30, 500)
    assert res.converged == bool(z["conv"])
    assert res.iterations == int(z["its"])
    assert np.linalg.norm(res.x - z["x"]) <= 1e-9 * np.linalg.norm(z["x"])
    r5 = O.gmres(J.matvec, b, pre.apply, 1e-10, 1e-14, 5, 500)
    assert r5.iterations == int(z["its5"]) and r5.converged == bool(z["conv5"])
    assert np.linalg.norm(r5.x - z["x5"]) <= 1e-9 * np.linalg.norm(z["x5"])
    rn = O.gmres(J.matvec, b, None, 1e-8, 1e-14, 30, 60)
    assert rn.iterations == int(z["itsn"]) and rn.converged == bool(z["convn"])
    assert np.linalg.norm(rn.x - z["xn"]) <= 1e-8 * np.linalg.norm(z["xn"])


NEWTON = {
    "a": ((12, 12), False, 1e-3, 4, 1, "ilu0", {}),
    "b": ((8, 8), False, 0.01, 2, 1, "lu", dict(reuse_factorization=False)),
    "c": ((8, 8), False, 1.0, 2, 1, "lu", dict(reuse_factorization=False)),
    "d": ((8, 8), False, 1e-2, 2, 1, "ilu0", dict(max_linear_iterations=1, gmres_restart=1)),
    "e": ((10, 8, 6), True, 1e-3, 4, 1, "ilu0", {}),
}


@pytest.mark.parametrize("tag", sorted(NEWTON))
def test_newton_matches_reference(tag):
    z = golden("newton.npz")
    counts, periodic, dt, nsub, ov, solver, kw = NEWTON[tag]
    m = O.Mesh(counts, tuple(1.0 for _ in counts), periodic)
    st = O.Step(m, CO, z[f"{tag}_u"], z[f"{tag}_v"], dt)
    pre = O.SchwarzOracle(O.decompose(m, nsub, ov), "ras-left", solver)
    trace = []
    x, rep = O.newton_solve(st, O.pack(z[f"{tag}_u"], z[f"{tag}_v"]), O.NewtonSettings(**kw), pre, trace)
    conv, nit, git, fac = (int(t) for t in z[f"{tag}_report"])
    assert rep.converged == bool(conv)
    assert rep.newton_iterations == nit
    assert abs(rep.gmres_iterations - git) <= 1
    assert rep.factorizations == fac
    assert (rep.reason or "") == str(z[f"{tag}_reason"])
    ref = z[f"{tag}_x"]
    assert np.linalg.norm(x - ref) <= 1e-8 * np.linalg.norm(ref)


def run_sim(tag):
    z = golden(f"sim_{tag}.npz")
    counts = tuple(int(c) for c in z["counts"])
    m = O.Mesh(counts, tuple(1.0 for _ in counts), bool(z["periodic"]))
    center, amp, dt, horizon, nsub, eta, max_steps = (float(t) for t in z["meta"])
    if eta < 0:
        eta = 1e4 if m.dim == 2 else 1e2
    u0, v0 = O.initial_fields(m, center, amp, 1234)
    if str(z["mode"]) == "fixed":
        ctl = O.Controller(dt, dt, eta, fixed_dt=dt)
    else:
        ctl = O.Controller(1e-4, 10.0, eta)
    status, rows, x, events = O.simulate(
        m, CO, u0, v0, ctl, horizon, int(nsub), 1, str(z["variant"]), str(z["solver"]),
        max_steps=None if max_steps < 0 else int(max_steps))
    return z, m, status, rows, x, ctl


def _compare_sim(z, m, status, rows, x, ctl):
    ref = z["rows"]
    assert status == str(z["status"])
    assert len(rows) == len(ref)
    got = np.array([[r.step, r.time, r.dt, r.energy, r.mass_u, r.max_abs_v, r.newton, r.gmres] for r in rows])
    np.testing.assert_array_equal(got[:, 0], ref[:, 0])
    np.testing.assert_allclose(got[:, 2], ref[:, 2], rtol=1e-10)          # accepted dt sequence
    np.testing.assert_allclose(got[:, 3], ref[:, 3], rtol=1e-10)          # energy
    np.testing.assert_allclose(got[:, 4], ref[:, 4], rtol=1e-12)          # mass
    np.testing.assert_array_equal(got[:, 6], ref[:, 6])                   # newton counts
    assert np.all(np.abs(got[:, 7] - ref[:, 7]) <= 2)                     # gmres counts
    assert ctl.divergence_count == int(z["divergences"])
    uref, vref = z["u"], z["v"]
    u, v = O.unpack(m, x)
    err = np.sqrt(np.sum((u - uref) ** 2 + (v - vref) ** 2) / np.sum(uref ** 2 + vref ** 2))
    assert err <= 1e-8


def test_simulate_config1_matches_reference():
    _compare_sim(*run_sim("c1"))


def test_simulate_adaptive_2d_matches_reference():
    _compare_sim(*run_sim("c2small"))


def test_simulate_adaptive_3d_neumann_matches_reference():
    _compare_sim(*run_sim("c3small"))


@pytest.mark.parametrize("tag", ["2d_neu", "2d_per", "2d_per4", "3d_neu", "3d_per"])
def test_fast_assembly_equals_reference_blocks(tag):
    z = golden(f"stencil_{tag}.npz")
    m = mesh_of(z)
    st = O.Step(m, CO, z["uo"], z["vo"], float(z["dt"]))
    ip, ix, bl = st.jacobian(O.pack(z["un"], z["vn"])).assemble_fast()
    assert np.array_equal(ip, z["J_indptr"])
    assert np.array_equal(ix, z["J_indices"])
    assert np.max(np.abs(bl - z["J_blocks"])) <= 1e-12 * np.max(np.abs(z["J_blocks"]))
