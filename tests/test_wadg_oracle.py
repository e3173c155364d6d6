"""Weight-adjusted (WADG) mass mode on the CPU oracle (config 4 of BASELINE.json).

WADG is the north star's reduced-storage update; the
reference stores the exact per-wedge lift instead, so there is no reference
output to pin against.  These tests pin the oracle's WADG restatement through
properties the method must have:
  * WADG == exact to round-off when J is constant (affine wedges);
  * on deformed wedges it is a different (consistent) method: small O(h^p) change;
  * energy stability in the Mtilde norm: dE/dt = u^T (S u + B) is the SAME
    number as for the exact operator (<= 0 upwind, == 0 central), measured by
    the exact central difference of the quadratic energy;
  * config 4 spectra on the perturbed 16-wedge mesh, N=2 (acceptance.cpp:103-131):
    exact and WADG upwind in the closed left half plane, central purely
    imaginary, lumped with eigenvalues of positive real part;
  * convergence at the same rate as the exact mode.
"""
import numpy as np
import pytest

import oracle_binding as ob
import paper_1607_03399_b200 as pdg


def rand(d, seed=7):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, d.total_dofs)


@pytest.mark.parametrize("degree", [1, 2, 3, 4, 5])
def test_wadg_equals_exact_for_constant_jacobian(degree):
    mesh = pdg.structured_hybrid_box(2, 2, 1, 1, (1.0, 2.0), (1.0, 4.0))
    de = pdg.build_discretization(mesh, degree)
    dw = pdg.build_discretization(mesh, degree, mass="wadg")
    u = rand(de)
    a, b = ob.rhs(de, u), ob.rhs(dw, u)
    assert np.abs(a - b).max() <= 1e-13 * np.abs(a).max()
    assert abs(ob.energy(de, u) - ob.energy(dw, u)) <= 1e-13 * ob.energy(de, u)


def test_wadg_is_a_small_change_on_deformed_wedges():
    mesh = pdg.spectra_mesh()
    de = pdg.build_discretization(mesh, 3)
    dw = pdg.build_discretization(mesh, 3, mass="wadg")
    s = pdg.make_initial_state(de)
    a, b = ob.rhs(de, s.u), ob.rhs(dw, s.u)
    rel = np.linalg.norm(a - b) / np.linalg.norm(a)
    assert 1e-6 < rel < 5e-2, rel


@pytest.mark.parametrize("mesh_name", ["spectra", "unstructured"])
def test_wadg_energy_rate_equals_exact(mesh_name):
    """E(u) quadratic => (E(u+h r) - E(u-h r)) / 2h is exactly u^T Mtilde r = u^T (S u + B)."""
    mesh = pdg.spectra_mesh() if mesh_name == "spectra" else pdg.make_family_mesh("unstructured", 0.5)
    u = None
    for flux in ("upwind", "central"):
        dw = pdg.build_discretization(mesh, 3, flux=flux, mass="wadg")
        de = pdg.build_discretization(mesh, 3, flux=flux)
        if u is None:
            u = rand(dw, 11)
        h = 1e-3
        rw, re = ob.rhs(dw, u), ob.rhs(de, u)
        rate_w = (ob.energy(dw, u + h * rw) - ob.energy(dw, u - h * rw)) / (2 * h)
        rate_e = (ob.energy(de, u + h * re) - ob.energy(de, u - h * re)) / (2 * h)
        scale = ob.energy(dw, u) * np.abs(rw).max()
        if flux == "central":
            assert abs(rate_w) <= 1e-12 * scale
        else:
            assert rate_w < 0.0
        assert abs(rate_w - rate_e) <= 1e-11 * scale


def _dense_operator(d):
    n = d.total_dofs
    A = np.empty((n, n))
    e = np.zeros(n)
    for k in range(n):
        e[k] = 1.0
        A[:, k] = ob.rhs(d, e, threads=1)
        e[k] = 0.0
    return A


@pytest.mark.slow
def test_config4_spectra_exact_wadg_lumped():
    """acceptance.cpp:103-131 criterion 3, extended with the WADG mode."""
    mesh = pdg.spectra_mesh()
    out = {}
    for mass in ("exact", "wadg", "lumped"):
        for flux in ("upwind", "central"):
            d = pdg.build_discretization(mesh, 2, flux=flux, mass=mass)
            assert d.total_dofs == 1152
            ev = np.linalg.eigvals(_dense_operator(d))
            out[(mass, flux)] = (ev.real.max(), np.abs(ev.real).max(), np.abs(ev).max())
    for mass in ("exact", "wadg"):
        re_u, _, abs_u = out[(mass, "upwind")]
        _, absre_c, abs_c = out[(mass, "central")]
        assert re_u <= 1e-10 * abs_u, (mass, re_u, abs_u)
        assert absre_c <= 1e-8 * abs_c, (mass, absre_c, abs_c)
    assert out[("lumped", "upwind")][0] > 0.0
    assert out[("lumped", "central")][0] > 0.0


def test_wadg_lserk_energy_never_increases_upwind():
    mesh = pdg.perturb_vertically(pdg.make_family_mesh("unstructured", 0.5), 0.3, 7)
    d = pdg.build_discretization(mesh, 3, mass="wadg")
    s = pdg.make_initial_state(d)
    dt = pdg.estimate_dt(d, 0.5)
    u = s.u
    e_prev = ob.energy(d, u)
    for _ in range(10):
        u = ob.lserk(d, u, dt, 5)
        e = ob.energy(d, u)
        assert e <= e_prev * (1 + 1e-12)
        e_prev = e


def test_wadg_convergence_rate_matches_exact():
    """Unstructured (deformed) family, N=2: WADG keeps the exact mode's accuracy."""
    errs = {"exact": [], "wadg": []}
    hs = [1.0, 0.5]
    for mass in errs:
        for h in hs:
            d = pdg.build_discretization(pdg.make_family_mesh("unstructured", h), 2, mass=mass)
            s = pdg.make_initial_state(d)
            dt = pdg.estimate_dt(d, 0.5)
            nsteps = int(np.ceil(0.5 / dt))
            u = ob.lserk(d, s.u, 0.5 / nsteps, nsteps)
            errs[mass].append(pdg.l2_error(d, u, 0.5))
    for k in range(len(hs)):
        assert abs(errs["wadg"][k] - errs["exact"][k]) <= 0.1 * errs["exact"][k], errs
    rate = lambda e: np.log(e[0] / e[1]) / np.log(hs[0] / hs[1])  # noqa: E731
    assert abs(rate(errs["wadg"]) - rate(errs["exact"])) <= 0.2, errs
