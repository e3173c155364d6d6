"""GPU parity of the weight-adjusted (WADG) wedge kernel against the CPU oracle.

The oracle restates WADG as (Mhat^-1 M_{1/J} Mhat^-1 M^{tri,k}) (x) I applied
to the exact rhs (oracle/hotpath.cpp); the kernel computes
Ltilde [K (rx Dr + sx Ds) U + ...] with Ltilde formed per wedge on the tensor
cores from j0, jr, js (csrc/cuda/wedge_wadg.cu).  Same tolerances as the exact
mode (tests/test_gpu_parity.py): rhs 1e-12 per field, 1e-10 after K steps,
energy 1e-12.
"""
import numpy as np
import pytest

import oracle_binding as ob
import paper_1607_03399_b200 as pdg
from test_gpu_parity import RHS_TOL, STEP_TOL, field_errors, random_state

pytestmark = pytest.mark.gpu

MESHES = {
    "spectra16": lambda: pdg.spectra_mesh(),
    "unstructured_h05": lambda: pdg.make_family_mesh("unstructured", 0.5),
    "hybrid_perturbed": lambda: pdg.perturb_vertically(
        pdg.structured_hybrid_box(2, 2, 2, 1, (1.0, 1.0), (1.0, 4.0)), 0.2, 3),
    "layers_media": lambda: pdg.perturb_vertically(
        pdg.layered_mesh(3, [-1.0, -0.2, 1.0], [2, 3], [(1.0, 1.0), (2.0, 4.0)]), 0.25, 9),
}


@pytest.mark.parametrize("mesh_name", sorted(MESHES))
@pytest.mark.parametrize("degree", [1, 2, 3, 4, 5, 6, 7])
def test_wadg_rhs_matches_oracle(mesh_name, degree):
    d = pdg.build_discretization(MESHES[mesh_name](), degree, mass="wadg")
    u = random_state(d, seed=degree)
    errs = field_errors(d, pdg.compute_rhs(d, u), ob.rhs(d, u))
    assert max(errs) <= (10 if degree >= 6 else 1) * RHS_TOL, errs


@pytest.mark.parametrize("flux", ["central", "custom"])
def test_wadg_flux_modes(flux):
    d = pdg.build_discretization(pdg.spectra_mesh(), 3, flux=flux, tau_p=0.7, tau_u=1.3, mass="wadg")
    u = random_state(d)
    errs = field_errors(d, pdg.compute_rhs(d, u), ob.rhs(d, u))
    assert max(errs) <= RHS_TOL, errs


def test_wadg_equals_exact_kernel_for_constant_jacobian():
    mesh = pdg.structured_hybrid_box(3, 3, 2, 1, (1.0, 2.0), (1.0, 4.0))
    de = pdg.build_discretization(mesh, 4)
    dw = pdg.build_discretization(mesh, 4, mass="wadg")
    u = random_state(de)
    a, b = pdg.compute_rhs(de, u), pdg.compute_rhs(dw, u)
    assert np.abs(a - b).max() <= 1e-12 * np.abs(a).max()


def test_wadg_without_host_lifts_is_identical():
    """Reduced storage end to end: no per-wedge operator on host or device."""
    mesh = pdg.perturb_vertically(pdg.structured_wedge_box(3), 0.3, 5)
    d1 = pdg.build_discretization(mesh, 3, mass="wadg")
    d2 = pdg.build_discretization(mesh, 3, mass="wadg", host_lifts=False)
    u = random_state(d1)
    assert np.array_equal(pdg.compute_rhs(d1, u), pdg.compute_rhs(d2, u))


@pytest.mark.parametrize("degree", [2, 5])
def test_wadg_phase_functions(degree):
    d = pdg.build_discretization(MESHES["hybrid_perturbed"](), degree, mass="wadg")
    u = random_state(d)
    ctx = d.device()
    ctx.set_state(u)
    want = ob.phase(d, 0, u, np.zeros(d.total_dofs))
    want = ob.phase(d, 1, u, want)
    ctx.phase("wedge_volume")
    ctx.phase("wedge_surface")
    got = ctx.get_rhs()
    nw = int(d.info.num_wedges)
    end = d.elem_offset()[nw]
    scale = np.abs(want[:end]).max()
    assert np.abs(got[:end] - want[:end]).max() <= RHS_TOL * scale


def test_wadg_lserk_steps_match_oracle():
    d = pdg.build_discretization(MESHES["unstructured_h05"](), 3, mass="wadg")
    s = pdg.make_initial_state(d)
    dt = pdg.estimate_dt(d, 0.5)
    ctx = d.device()
    ctx.set_state(s.u)
    ctx.step(dt, 100)
    got = ctx.get_state()
    want = ob.lserk(d, s.u, dt, 100)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) <= STEP_TOL


@pytest.mark.parametrize("degree", [2, 3, 7])
def test_wadg_energy_matches_oracle(degree):
    d = pdg.build_discretization(MESHES["hybrid_perturbed"](), degree, mass="wadg")
    u = random_state(d)
    e_gpu, e_orc = pdg.compute_energy(d, u), ob.energy(d, u)
    assert abs(e_gpu - e_orc) <= 1e-12 * abs(e_orc)


def test_wadg_run_simulation_energy_never_increases():
    d = pdg.build_discretization(MESHES["layers_media"](), 3, mass="wadg")
    s = pdg.make_initial_state(d)
    res = pdg.run_simulation(d, s, pdg.RunOptions(final_time=0.5))
    assert res.max_energy_increase <= 1e-10 * res.initial_energy
    assert res.final_energy < res.initial_energy


def test_wadg_spectrum_on_gpu_operator():
    """Config 4 on the device operator: upwind spectrum in the closed left half plane."""
    d = pdg.build_discretization(pdg.spectra_mesh(), 2, mass="wadg")
    ctx = d.device()
    n = d.total_dofs
    A = np.empty((n, n))
    e = np.zeros(n)
    for k in range(n):
        e[k] = 1.0
        A[:, k] = ctx.rhs(e)
        e[k] = 0.0
    ev = np.linalg.eigvals(A)
    assert ev.real.max() <= 1e-10 * np.abs(ev).max()
