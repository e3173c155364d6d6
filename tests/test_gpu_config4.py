"""BASELINE configs[3] (ii) / SURVEY 8(d) row 4: the long deformed-layer run.

The reference's "layers" mesh kind with a sine interface (config.cpp:152-178:
sine:z0:amp:kx:ky = z0 + amp sin(pi kx x) cos(pi ky y)) on the n = 32 surface,
perturbed vertically (perturb_vertically(0.3, 7), mesh.cpp:327-333), so J
varies inside every wedge; 1000 LSERK45 steps with the energy logged every 10
steps on the GPU.  Exact and weight-adjusted mass: the upwind energy (in each
scheme's own norm) never grows; the exact-mass run equals the CPU oracle after
the 1000 steps."""
import os

import numpy as np
import pytest

import oracle_binding as ob
import paper_1607_03399_b200 as pdg
from parity_util import rel_l2

pytestmark = pytest.mark.gpu


def sine_layers_mesh(n=32, sublayers=(4, 4)):
    xy, tris = pdg.structured_surface(n)
    x, y = xy[:, 0], xy[:, 1]
    mid = 0.0 + 0.2 * np.sin(np.pi * 1.0 * x) * np.cos(np.pi * 1.0 * y)  # sine:0:0.2:1:1
    layers = [pdg.LayerSpec(np.full(len(x), -1.0), mid, sublayers[0], (1.0, 1.0)),
              pdg.LayerSpec(mid, np.full(len(x), 1.0), sublayers[1], (1.0, 2.25))]
    return pdg.perturb_vertically(pdg.stack_layers(xy, tris, layers), 0.3, 7)


@pytest.mark.parametrize("mass,degree", [("exact", 2), ("wadg", 2), ("exact", 3), ("wadg", 3)])
def test_long_deformed_layer_run(mass, degree):
    m = sine_layers_mesh()
    assert m.num_wedges() == 2 * 32 * 32 * 8
    d = pdg.build_discretization(m, degree, mass=mass, threads=os.cpu_count() or 4)
    s = pdg.make_initial_state(d, "gaussian", [0.3, 0.0, 0.0, 0.2])
    u0 = s.u.copy()
    dt = pdg.estimate_dt(d, 0.5)
    res = pdg.run_simulation(d, s, pdg.RunOptions(final_time=1000 * dt, fixed_dt=dt, energy_interval=10 * dt))
    assert res.steps == 1000
    log = res.energy_log
    assert len(log) == 101
    e = log[:, 1]
    assert np.all(np.diff(e) <= 1e-10 * e[0]), np.diff(e).max()
    assert e[-1] < e[0]
    if mass == "exact" and degree == 2:
        want = ob.lserk(d, u0, dt, 1000, threads=os.cpu_count() or 4)
        assert rel_l2(s.u, want) <= 1e-10
