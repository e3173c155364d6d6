"""GPU vs oracle at the parity sizes SURVEY.md 8(d) names for the benchmarked configs.

* configs[1] (the order sweep, 1e6 layered wedges): its 1/100-size copy
  (n=10 surface x the same 15/15/20 sublayers = 10,000 wedges) at N = 1..7, in
  exact mode and in the weight-adjusted mode on the same mesh perturbed
  vertically (varying J, configs[3]'s update): one RHS and 3 LSERK45 steps.
  The kernels hand work out through a global ticket counter; the launch record
  proves every team looped over several tickets, so the cross-element
  machinery (double-buffered TMA stages, parity flux buffers, dropped end
  barriers, ticket batches) is what the oracle checks here.
* the full 1e6-wedge N = 5 mesh itself: one RHS against the oracle.
* configs[2] at its parity mesh structured_hybrid_box(4,4,2,2), N = 4.
* row f2: the assembled device operator against oracle columns.
Tolerances as tests/test_gpu_parity.py: RHS max-abs <= 1e-12 x max|rhs| per
field, K steps relative L2 <= 1e-10 (FP64; the GPU sums in another order).
"""
import os

import numpy as np
import pytest

import oracle_binding as ob
import paper_1607_03399_b200 as pdg
from parity_util import config2_mesh, field_errors, rel_l2

pytestmark = pytest.mark.gpu

RHS_TOL = 1e-12
STEP_TOL = 1e-10
THREADS = os.cpu_count() or 4

_MESHES = {}


def mesh(kind):
    if kind not in _MESHES:
        if kind == "copy100":  # the 1/100-size copy of configs[1]
            _MESHES[kind] = config2_mesh(10, (15, 15, 20))
        elif kind == "copy100_deformed":
            _MESHES[kind] = pdg.perturb_vertically(config2_mesh(10, (15, 15, 20)), 0.3, 7)
        elif kind == "wide":  # 120,000 wedges: several tickets per CTA for the low-order kernels
            _MESHES[kind] = config2_mesh(100, (2, 2, 2))
    return _MESHES[kind]


def check_multi_ticket(ctx, kind="wedge", min_ratio=2.0):
    li = ctx.launch_info()[kind]
    assert li["launched"] == 1, li
    assert li["tickets"] >= min_ratio * li["teams"], li
    return li


@pytest.mark.parametrize("mass", ["exact", "wadg"])
@pytest.mark.parametrize("degree", [1, 2, 3, 4, 5, 6, 7])
def test_config2_copy_rhs_and_steps(degree, mass):
    m = mesh("copy100" if mass == "exact" else "copy100_deformed")
    assert m.num_wedges() == 10_000
    d = pdg.build_discretization(m, degree, mass=mass, threads=THREADS)
    u = np.random.default_rng(100 + degree).uniform(-1.0, 1.0, d.total_dofs)
    ctx = d.device()
    got = ctx.rhs(u)
    want = ob.rhs(d, u, threads=THREADS)
    errs = field_errors(d, got, want)
    assert max(errs) <= RHS_TOL, errs
    if degree >= 4:
        check_multi_ticket(ctx)
    # 3 LSERK steps of a smooth state (configs[1]'s Gaussian pulse) plus a rough one
    dt = pdg.estimate_dt(d, 0.5)
    for u0 in (pdg.make_initial_state(d, "gaussian", [0.25, 0.0, 0.0, 0.0]).u, u):
        ctx.set_state(u0)
        ctx.step(dt, 3)
        if degree >= 4:
            check_multi_ticket(ctx)
        rel = rel_l2(ctx.get_state(), ob.lserk(d, u0, dt, 3, threads=THREADS))
        assert rel <= STEP_TOL, rel


@pytest.mark.parametrize("mass", ["exact", "wadg"])
@pytest.mark.parametrize("degree", [1, 2, 3])
def test_low_order_kernels_multi_ticket(degree, mass):
    """The CUDA-core kernels (N <= 3) take chunks of 128/NT wedges per ticket; on
    120k wedges every CTA loops over several chunks (double-buffered cp.async)."""
    m = mesh("wide")
    if mass == "wadg":
        m = pdg.perturb_vertically(m, 0.3, 7)
    d = pdg.build_discretization(m, degree, mass=mass, threads=THREADS)
    u = np.random.default_rng(7 + degree).uniform(-1.0, 1.0, d.total_dofs)
    ctx = d.device()
    errs = field_errors(d, ctx.rhs(u), ob.rhs(d, u, threads=THREADS))
    assert max(errs) <= RHS_TOL, errs
    li = check_multi_ticket(ctx)
    dt = pdg.estimate_dt(d, 0.5)
    ctx.set_state(u)
    ctx.step(dt, 2)
    assert rel_l2(ctx.get_state(), ob.lserk(d, u, dt, 2, threads=THREADS)) <= STEP_TOL, li


def test_full_size_config2_rhs_n5():
    """The benchmark mesh itself (1e6 wedges, N = 5, 504M DOFs): one RHS vs the oracle."""
    m = config2_mesh(100, (15, 15, 20))
    assert m.num_wedges() == 1_000_000
    d = pdg.build_discretization(m, 5, threads=THREADS)
    assert d.total_dofs == 504_000_000
    u = np.random.default_rng(2016).uniform(-1.0, 1.0, d.total_dofs)
    ctx = pdg.DeviceContext(d)
    got = ctx.rhs(u)
    li = check_multi_ticket(ctx, min_ratio=10.0)
    ctx.close()
    want = ob.rhs(d, u, threads=THREADS)
    errs = field_errors(d, got, want)
    assert max(errs) <= RHS_TOL, (errs, li)


def test_config3_parity_mesh_n4():
    """configs[2]'s parity mesh: structured_hybrid_box(4,4,2,2), wedge media (1,1),
    tet media (1,4), N = 4 (both the wedge DMMA and the tet DMMA kernels)."""
    m = pdg.structured_hybrid_box(4, 4, 2, 2, (1.0, 1.0), (1.0, 4.0))
    d = pdg.build_discretization(m, 4)
    u = np.random.default_rng(34).uniform(-1.0, 1.0, d.total_dofs)
    ctx = d.device()
    errs = field_errors(d, ctx.rhs(u), ob.rhs(d, u))
    assert max(errs) <= RHS_TOL, errs
    li = ctx.launch_info()
    assert li["wedge"]["launched"] == 1 and li["tet"]["launched"] == 1, li
    dt = pdg.estimate_dt(d, 0.5)
    for u0 in (u, pdg.make_initial_state(d, "gaussian", [0.25, 0.0, 0.0, 0.0]).u):
        ctx.set_state(u0)
        ctx.step(dt, 3)
        assert rel_l2(ctx.get_state(), ob.lserk(d, u0, dt, 3)) <= STEP_TOL


def test_wedge_only_mesh_launches_no_tet_kernel():
    """gpu_launches counts real launches: on a wedge-only mesh the (empty) tet
    stage launches nothing and records no timing events."""
    d = pdg.build_discretization(mesh("copy100"), 3)
    ctx = pdg.DeviceContext(d, flags=pdg.capi.CTX_TIMING)
    ctx.set_state(np.zeros(d.total_dofs))
    ctx.step(1e-3, 2)
    kt = ctx.kernel_times(reset=True)
    assert kt["wedge_launches"] == 10 and kt["tet_launches"] == 0, kt
    assert ctx.launch_info()["tet"]["launched"] == 0
    ctx.close()


@pytest.mark.parametrize("mass", ["exact", "wadg", "lumped"])
def test_assembled_operator_matches_oracle_columns(mass):
    """f2 (analysis.cpp:12-40): every column of the device-assembled operator
    equals the oracle's rhs of the unit vector (the 1152-DOF spectra mesh)."""
    d = pdg.build_discretization(pdg.spectra_mesh(), 2, mass=mass)
    n = d.total_dofs
    assert n == 1152
    A = pdg.assemble_global(d)
    want = np.empty((n, n), order="F")
    e = np.zeros(n)
    for j in range(n):
        e[j] = 1.0
        want[:, j] = ob.rhs(d, e, threads=1)
        e[j] = 0.0
    scale = np.abs(want).max()
    assert np.abs(A - want).max() <= RHS_TOL * scale
    # structure: an operator column only touches its element and the face neighbours
    assert np.array_equal(A == 0.0, want == 0.0) or np.abs(A[want == 0.0]).max() <= 1e-14 * scale


def test_rhs_bitwise_deterministic_config2_copy():
    """test_solver.cpp:202-212 (bitwise thread-count invariance) on the device:
    run to run and context to context the RHS and 3 steps are bitwise equal."""
    d = pdg.build_discretization(mesh("copy100"), 5)
    u = np.random.default_rng(3).uniform(-1.0, 1.0, d.total_dofs)
    outs = []
    for _ in range(2):
        ctx = pdg.DeviceContext(d)
        r = ctx.rhs(u)
        ctx.set_state(u)
        ctx.step(pdg.estimate_dt(d, 0.5), 3)
        outs.append((r, ctx.get_state()))
        ctx.close()
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
