"""Edge cases of the device path against the CPU oracle: single elements,
wedge-only / tet-only meshes, the high-order CUDA-core tet kernel (N >= 6),
WADG on hybrid meshes (tets stay exact), the phase API in WADG mode, and
the interior/boundary stage split on an unpartitioned context."""
import ctypes as C

import numpy as np
import pytest

import oracle_binding as ob
import paper_1607_03399_b200 as pdg
from paper_1607_03399_b200.capi import check, lib
from test_gpu_parity import RHS_TOL, field_errors, random_state

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mesh_fn", [lambda: pdg.structured_hybrid_box(1, 1, 1, 0),
                                     lambda: pdg.structured_hybrid_box(1, 1, 0, 1)])
@pytest.mark.parametrize("degree", [1, 4, 7])
def test_tiny_meshes(mesh_fn, degree):
    d = pdg.build_discretization(mesh_fn(), degree)
    u = random_state(d, seed=degree)
    errs = field_errors(d, pdg.compute_rhs(d, u), ob.rhs(d, u))
    assert max(errs) <= 10 * RHS_TOL, errs


@pytest.mark.parametrize("degree", [6, 7])
def test_high_order_tets_simt_kernel(degree):
    d = pdg.build_discretization(pdg.structured_hybrid_box(2, 2, 1, 2, (1.0, 1.0), (1.0, 4.0)), degree)
    u = random_state(d, seed=degree)
    errs = field_errors(d, pdg.compute_rhs(d, u), ob.rhs(d, u))
    assert max(errs) <= 10 * RHS_TOL, errs
    dt = pdg.estimate_dt(d, 0.5)
    ctx = d.device()
    ctx.set_state(u)
    ctx.step(dt, 3)
    want = ob.lserk(d, u, dt, 3)
    assert np.linalg.norm(ctx.get_state() - want) / np.linalg.norm(want) <= 1e-10


@pytest.mark.parametrize("degree", [2, 4])
def test_wadg_hybrid_with_tets(degree):
    mesh = pdg.perturb_vertically(pdg.structured_hybrid_box(2, 2, 2, 1, (1.0, 1.0), (1.0, 4.0)), 0.2, 11)
    d = pdg.build_discretization(mesh, degree, mass="wadg")
    u = random_state(d, seed=3)
    errs = field_errors(d, pdg.compute_rhs(d, u), ob.rhs(d, u))
    assert max(errs) <= RHS_TOL, errs
    ctx = d.device()
    ctx.set_state(u)
    for which, code in (("tet", 2),):
        want = ob.phase(d, code, u, np.zeros(d.total_dofs))
        want = ob.phase(d, code + 1, u, want)
        ctx.phase(f"{which}_volume")
        ctx.phase(f"{which}_surface")
        got = ctx.get_rhs()
        nw = int(d.info.num_wedges)
        sl = slice(d.elem_offset()[nw], d.elem_offset()[-1])
        assert np.abs(got[sl] - want[sl]).max() <= RHS_TOL * np.abs(want[sl]).max()


def test_stage_parts_on_unpartitioned_context():
    """Unpartitioned: every element is interior, part 1 computes all, part 2 none."""
    d = pdg.build_discretization(pdg.structured_hybrid_box(2, 2, 1, 1), 3)
    u = random_state(d)
    dt = pdg.estimate_dt(d, 0.5)
    a = d.device()
    a.set_state(u)
    a.step(dt, 1)
    b = d.device()
    b.set_state(u)
    for s in range(5):
        check(lib().pdg_step_stage_part(b.handle, dt, s, 1))
        check(lib().pdg_step_stage_part(b.handle, dt, s, 2))
    assert np.array_equal(a.get_state(), b.get_state())
    counts = (C.c_int64 * 6)()
    check(lib().pdg_partition_counts(b.handle, counts))
    assert counts[4] == counts[0] and counts[5] == counts[1]
