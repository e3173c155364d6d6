"""AB3 integrator (TimeStepper::step, proj/src/solver.cpp:559-581).

CPU: the oracle restatement -- two LSERK45 bootstrap steps, then
u += dt/12 (23 f_n - 16 f_{n-1} + 5 f_{n-2}); GPU: pdg_step_ab3 / run_simulation
with integrator ab3 against it.
"""
import numpy as np
import pytest

import oracle_binding as ob
import paper_1607_03399_b200 as pdg


def test_ab3_bootstrap_is_lserk():
    d = pdg.build_discretization(pdg.structured_hybrid_box(2, 2, 1, 1), 2)
    s = pdg.make_initial_state(d)
    dt = 0.25 * pdg.estimate_dt(d, 0.5)
    assert np.array_equal(ob.ab3(d, s.u, dt, 2), ob.lserk(d, s.u, dt, 2, parallel_update=False))


def test_ab3_accuracy_matches_lserk():
    """Structured h=0.5, N=3 to t=0.5: the spatial error dominates both integrators."""
    d = pdg.build_discretization(pdg.make_family_mesh("structured", 0.5), 3)
    s = pdg.make_initial_state(d)
    T = 0.5
    n_rk = int(np.ceil(T / pdg.estimate_dt(d, 0.5)))
    n_ab = int(np.ceil(T / (0.25 * pdg.estimate_dt(d, 0.5))))
    e_rk = pdg.l2_error(d, ob.lserk(d, s.u, T / n_rk, n_rk), T)
    e_ab = pdg.l2_error(d, ob.ab3(d, s.u, T / n_ab, n_ab), T)
    assert abs(e_ab - e_rk) <= 0.05 * e_rk, (e_ab, e_rk)


@pytest.mark.gpu
@pytest.mark.parametrize("mass", ["exact", "wadg"])
def test_gpu_ab3_matches_oracle(mass):
    mesh = pdg.perturb_vertically(pdg.structured_hybrid_box(2, 2, 2, 1, (1.0, 1.0), (1.0, 4.0)), 0.2, 3)
    d = pdg.build_discretization(mesh, 3, mass=mass)
    s = pdg.make_initial_state(d)
    dt = 0.25 * pdg.estimate_dt(d, 0.5)
    ctx = d.device()
    ctx.set_state(s.u)
    t = ctx.step(dt, 40, integrator="ab3")
    assert abs(t - 40 * dt) <= 1e-14
    got = ctx.get_state()
    want = ob.ab3(d, s.u, dt, 40)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-10


@pytest.mark.gpu
def test_gpu_ab3_history_resets_with_state():
    d = pdg.build_discretization(pdg.structured_wedge_box(2), 2)
    s = pdg.make_initial_state(d)
    dt = 0.25 * pdg.estimate_dt(d, 0.5)
    ctx = d.device()
    ctx.set_state(s.u)
    ctx.step(dt, 5, integrator="ab3")
    ctx.set_state(s.u)  # new state: the bootstrap runs again
    ctx.step(dt, 3, integrator="ab3")
    want = ob.ab3(d, s.u, dt, 3)
    got = ctx.get_state()
    assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-10


@pytest.mark.gpu
def test_gpu_run_simulation_ab3():
    d = pdg.build_discretization(pdg.spectra_mesh(), 3)
    s = pdg.make_initial_state(d)
    res = pdg.run_simulation(d, s, pdg.RunOptions(final_time=0.3, integrator="ab3"))
    dt0 = 0.25 * pdg.estimate_dt(d, 0.5)
    assert res.steps == int(np.ceil(0.3 / dt0 - 1e-12))
    assert res.max_energy_increase <= 1e-10 * res.initial_energy
    s2 = pdg.make_initial_state(d)
    want = ob.ab3(d, s2.u, res.dt, res.steps)
    assert np.linalg.norm(s.u - want) / np.linalg.norm(want) <= 1e-10
