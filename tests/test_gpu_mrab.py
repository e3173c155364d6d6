"""Multi-rate AB3 on the device (pdg_step_mrab) against the
oracle restatement (oracle/hotpath.cpp mrab_steps) on the same rate levels."""
import numpy as np
import pytest

import oracle_binding as ob
import paper_1607_03399_b200 as pdg
from mrab_util import levels, two_level_mesh
from parity_util import config2_mesh, rel_l2

pytestmark = pytest.mark.gpu


def mrab_ctx(d, L=3):
    return pdg.DeviceContext(d, flags=pdg.capi.CTX_MRAB_LEVELS(L))


@pytest.mark.parametrize("mesh_fn,degree", [(two_level_mesh, 2), (lambda: config2_mesh(4, (3, 3, 4)), 3),
                                            (lambda: pdg.perturb_vertically(config2_mesh(4, (3, 3, 4)), 0.3, 7), 4),
                                            (lambda: pdg.structured_hybrid_box(3, 3, 2, 2, (1.0, 1.0), (1.0, 4.0)), 3)])
def test_levels_and_steps_match_oracle(mesh_fn, degree):
    d = pdg.build_discretization(mesh_fn(), degree)
    ctx = mrab_ctx(d)
    lev, nlev = ctx.mrab_levels()
    assert np.array_equal(lev, levels(d, 3)) and nlev == lev.max() + 1
    u0 = np.random.default_rng(degree).uniform(-1, 1, d.total_dofs)
    dt = 0.25 * pdg.estimate_dt(d, 0.5)
    ctx.set_state(u0)
    t = ctx.step(dt, 6, integrator="mrab")
    assert abs(t - 6 * dt * (1 << (nlev - 1))) <= 1e-14
    want = ob.mrab(d, u0, lev, nlev, dt, 6)
    assert rel_l2(ctx.get_state(), want) <= 1e-10
    ctx.close()


def test_single_level_is_device_ab3_bitwise():
    d = pdg.build_discretization(pdg.structured_wedge_box(2), 3)
    ctx = mrab_ctx(d)
    assert ctx.mrab_levels()[1] == 1
    u0 = pdg.make_initial_state(d).u
    dt = 0.25 * pdg.estimate_dt(d, 0.5)
    ctx.set_state(u0)
    ctx.step(dt, 9, integrator="mrab")
    ref = d.device()
    ref.set_state(u0)
    ref.step(dt, 9, integrator="ab3")
    assert np.array_equal(ctx.get_state(), ref.get_state())
    ctx.close()


def test_mrab_third_order_and_run_simulation():
    """third order against expm(A T) on the two-level mesh; run_simulation with
    integrator="mrab" (macro steps of 2^L AB3 steps) keeps upwind energy bounded."""
    from scipy.linalg import expm
    d = pdg.build_discretization(two_level_mesh(), 2)
    A = pdg.assemble_global(d)
    u0 = pdg.make_initial_state(d).u
    T = 0.5
    exact = expm(A * T) @ u0
    ctx = mrab_ctx(d)
    nlev = ctx.mrab_levels()[1]
    assert nlev == 2
    dt0 = 0.25 * pdg.estimate_dt(d, 0.5)
    errs = []
    for k in range(3):
        nm = int(np.ceil(T / (2 * dt0 / (1 << k))))
        ctx.set_state(u0)
        ctx.step(T / nm / 2, nm, integrator="mrab")
        errs.append(np.linalg.norm(ctx.get_state() - exact))
    order = np.log2(errs[0] / errs[2]) / 2.0
    assert abs(order - 3.0) <= 0.3, (order, errs)
    ctx.close()
    s = pdg.make_initial_state(d)
    res = pdg.run_simulation(d, s, pdg.RunOptions(final_time=2.0, integrator="mrab"))
    assert res.final_energy <= res.initial_energy * (1 + 1e-10)
    assert abs(s.time - 2.0) <= 1e-12


def test_config2_copy_mrab_rhs_savings():
    """On the configs[1] layering (c = 1, 2, 1.5 with equal sublayer thickness)
    the kappa = 1 layer is level 1: 30% of the wedges evaluate their rhs every
    other fine step; parity with the oracle on the 1/100-size copy."""
    d = pdg.build_discretization(config2_mesh(10, (15, 15, 20)), 3)
    ctx = mrab_ctx(d)
    lev, nlev = ctx.mrab_levels()
    assert nlev == 2 and abs((lev == 1).mean() - 0.3) < 1e-12
    u0 = pdg.make_initial_state(d, "gaussian", [0.25, 0.0, 0.0, 0.0]).u
    dt = 0.25 * pdg.estimate_dt(d, 0.5)
    ctx.set_state(u0)
    ctx.step(dt, 5, integrator="mrab")
    assert rel_l2(ctx.get_state(), ob.mrab(d, u0, lev, nlev, dt, 5, threads=8)) <= 1e-10
    ctx.close()
