"""The C++ drop-in shim on the GPU: tests/cpp/test_shim.cpp (built into
paper_1607_03399_b200/_lib/test_shim, linked against the product only) calls
prismdg::compute_rhs / the phase functions / compute_energy / step (LSERK45 and
AB3 TimeSteppers) / run_simulation exactly as the reference's own C++ callers do
(proj/include/prismdg/solver.hpp:61-149); its outputs are checked here against
the CPU oracle on the same discretization (same generator, bit-identical mesh).
Also: a discretization ingested from arrays (pdg_disc_from_arrays) runs on the
device bitwise like the one it was exported from."""
import os
import subprocess

import numpy as np
import pytest

import oracle_binding as ob
import paper_1607_03399_b200 as pdg
from parity_util import field_errors, rel_l2

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = os.path.join(ROOT, "paper_1607_03399_b200", "_lib", "test_shim")


@pytest.fixture(scope="module")
def shim_out(tmp_path_factory):
    out = tmp_path_factory.mktemp("shim")
    r = subprocess.run([SHIM, str(out)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    return lambda name: np.fromfile(out / f"{name}.bin", dtype=np.float64)


@pytest.fixture(scope="module")
def disc():
    return pdg.build_discretization(pdg.structured_hybrid_box(2, 2, 1, 1, (1.0, 1.0), (1.0, 4.0)), 3)


def test_shim_rhs_phases_energy(shim_out, disc):
    u = shim_out("u")
    want = ob.rhs(disc, u)
    assert max(field_errors(disc, shim_out("rhs"), want)) <= 1e-12
    ph = np.zeros_like(u)
    for which in range(4):
        ob.phase(disc, which, u, ph)
    assert max(field_errors(disc, shim_out("phases"), ph)) <= 1e-12
    e = shim_out("energy")[0]
    assert abs(e - ob.energy(disc, u)) <= 1e-12 * ob.energy(disc, u)


def test_shim_time_steppers(shim_out, disc):
    u = shim_out("u")
    dt = pdg.estimate_dt(disc, 0.5)
    assert rel_l2(shim_out("lserk3"), ob.lserk(disc, u, dt, 3)) <= 1e-10
    assert rel_l2(shim_out("ab3_5"), ob.ab3(disc, u, 0.25 * dt, 5)) <= 1e-10


def test_shim_run_simulation(shim_out, disc):
    s = pdg.make_initial_state(disc)
    u, t, res = ob.run(disc, s.u, 0.0, 0.25, cfl=0.5, energy_interval=0.05)
    got = shim_out("run_result")
    steps, dt, final_time, e0, e1 = got[:5]
    assert int(steps) == int(res["steps"]) and dt == res["dt"]
    assert abs(final_time - 0.25) <= 1e-12 and got[7] == final_time
    assert abs(e0 - res["initial_energy"]) <= 1e-12 * e0 and abs(e1 - res["final_energy"]) <= 1e-10 * e0
    assert int(got[6]) == 1 + 5  # initial + every 0.05
    assert rel_l2(shim_out("run_state"), u) <= 1e-10


@pytest.mark.parametrize("degree", [2, 5])
def test_ingested_discretization_runs_on_device(degree):
    d = pdg.build_discretization(pdg.structured_hybrid_box(3, 3, 2, 1, (1.0, 1.0), (1.0, 4.0)), degree)
    d2 = pdg.discretization_from_arrays(pdg.export_arrays(d))
    u = np.random.default_rng(degree).uniform(-1, 1, d.total_dofs)
    r1, r2 = pdg.compute_rhs(d, u), pdg.compute_rhs(d2, u)
    assert np.array_equal(r1, r2)
    assert max(field_errors(d2, r2, ob.rhs(d2, u))) <= 1e-12
    c1, c2 = d.device(), d2.device()
    c1.set_state(u)
    c2.set_state(u)
    c1.step(1e-3, 2)
    c2.step(1e-3, 2)
    assert np.array_equal(c1.get_state(), c2.get_state())
    assert c1.energy() == c2.energy()
