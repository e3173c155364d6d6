"""Multi-rate AB3 (the paper's integrator) on
the CPU oracle: with one rate level it is the reference's AB3 (solver.cpp:
559-581) bit for bit, and on a two-level mesh it converges at third order to
the exact propagator of the assembled operator."""
import numpy as np
import pytest

import oracle_binding as ob
import paper_1607_03399_b200 as pdg
from mrab_util import levels, two_level_mesh


def test_single_level_is_ab3_bitwise():
    d = pdg.build_discretization(pdg.structured_hybrid_box(2, 2, 1, 1), 2)
    u = pdg.make_initial_state(d).u
    dt = 0.25 * pdg.estimate_dt(d, 0.5)
    lev = np.zeros(d.num_elements(), dtype=np.int32)
    assert np.array_equal(ob.mrab(d, u, lev, 1, dt, 7), ob.ab3(d, u, dt, 7))


def test_two_level_mesh_levels():
    d = pdg.build_discretization(two_level_mesh(), 2)
    lev = levels(d, 3)
    nw = int(d.info.num_wedges)
    assert set(lev.tolist()) == {0, 1}
    # the fast (kappa = 4) layer is level 0, the slow one level 1
    assert np.all(lev[: nw // 2] == 1) and np.all(lev[nw // 2:] == 0)


def test_mrab_third_order_vs_exact_propagator():
    from scipy.linalg import expm
    d = pdg.build_discretization(two_level_mesh(), 2)
    n = d.total_dofs
    A = np.empty((n, n))
    e = np.zeros(n)
    for j in range(n):
        e[j] = 1.0
        A[:, j] = ob.rhs(d, e, threads=1)
        e[j] = 0.0
    lev = levels(d, 3)
    u0 = pdg.make_initial_state(d).u
    T = 0.5
    exact = expm(A * T) @ u0
    dt0 = 0.25 * pdg.estimate_dt(d, 0.5)
    errs = []
    for k in range(3):
        macro = 2 * dt0 / (1 << k)       # 2 fine steps per macro step
        nm = int(np.ceil(T / macro))
        got = ob.mrab(d, u0, lev, 2, T / nm / 2, nm, threads=2)
        errs.append(np.linalg.norm(got - exact))
    order = np.log2(errs[0] / errs[2]) / 2.0
    assert abs(order - 3.0) <= 0.3, (order, errs)
